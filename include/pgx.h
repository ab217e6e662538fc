/*
 * pgx.h -- C ABI of libpgx.so, the B200 (sm_100a) superstep engine that
 * replaces the hot path of the reference `pregelite` package.
 *
 * The reference reaches its hot path only through
 *     pregelite.run(graph, program, config) -> RunReport
 *         (/root/reference/pkg/src/pregelite/engine.py:201-204)
 * whose body is `_Executor.run` (engine.py:255-316).  Each entry point
 * below names the reference interface it replaces.  The Python host mirror
 * (paper_2010_01542_b200/engine.py) binds these with ctypes; INTEGRATION.md
 * shows the binding a maintainer of the reference would add.
 *
 * Conventions
 *   - plain pointers and sizes only; every pointer argument that is not
 *     marked "host" is a device pointer owned by the caller (the library
 *     borrows it for the call and never frees it);
 *   - calls are stream-ordered and asynchronous unless marked "syncs";
 *     `stream` is a cudaStream_t passed as uintptr_t (0 = legacy default);
 *   - return 0 on success or a negative PGX_E* code; pgx_last_error()
 *     returns a thread-local message for the last failure.  The Python
 *     side maps PGX_EINVAL to pregelite.ConfigError and everything else to
 *     pregelite.ExecutionError (engine.py:277-280, 477-490).
 *   - vertex ids are int32 (graph.py:143 default id dtype) and row offsets
 *     are int32 on the device, so n < 2^31 and m < 2^31 (C5: m = 1.84e9).
 */
#ifndef PGX_H
#define PGX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PGX_ABI_VERSION 6

#define PGX_OK 0
#define PGX_EINVAL (-1)   /* bad argument / unsupported configuration */
#define PGX_ECUDA (-2)    /* CUDA runtime or kernel failure */
#define PGX_ENOMEM (-3)   /* workspace too small */

/* apps (the three lowered vertex programs, algorithms.py:27-152) */
#define PGX_APP_PAGERANK 0
#define PGX_APP_CC 1
#define PGX_APP_SSSP 2
#define PGX_APP_PAGERANK_PULL 3   /* pagerank in the reference's pull mode */

/* combine operators (mailbox.py:58-70 min_combine / sum_combine) */
#define PGX_OP_MIN_U32 0
#define PGX_OP_SUM_F64 1

/*
 * Per-run statistics written by the device (int64 words):
 *   stats[0] superstep_count        (RunReport.superstep_count)
 *   stats[1] hit_superstep_cap      (RunReport.hit_superstep_cap)
 *   stats[2] persistent CTAs used
 *   stats[3] kernel start, %globaltimer ns
 *   then PGX_STAT_FIELDS words per superstep s at stats + PGX_STAT_HDR +
 *   s * PGX_STAT_FIELDS:
 *     [0] active_count   (SuperstepStats.active_count, engine.py:284-286)
 *     [1] messages_sent  (SuperstepStats.messages_sent)
 *     [2] edges traversed by this superstep's senders (for GTEPS)
 *     [3] senders with out-degree > 0 (#F_s)
 *     [4] recipients of this superstep's messages (R_s)
 *     [5] superstep end, %globaltimer ns
 *     [6] vertices that computed a new value and sent (broadcasters)
 *     [7] scatter start (end of this superstep's apply), %globaltimer ns
 */
#define PGX_STAT_HDR 4
#define PGX_STAT_FIELDS 8

int pgx_abi_version(void);
const char *pgx_last_error(void);

/* process-wide tuning knobs (A/B experiments; defaults are shipped) */
#define PGX_OPT_READ_FILTER 0   /* 1: skip the atomic when min(old,msg)==old */
#define PGX_OPT_CTAS_PER_SM 1   /* persistent CTAs per SM, 0 = occupancy max */
#define PGX_OPT_CAS_LOOP 2      /* ablation: CAS retry loop per message (lock-style) */
#define PGX_OPT_VERTEX_SCHED 3  /* ablation: one thread per sender (no edge balance) */
#define PGX_OPT_LAYOUT 4        /* ablation: PGX_LAYOUT_* of the CC/SSSP vertex state */
#define PGX_OPT_SEG_MIN_EDGES 5 /* segmented scatter when a superstep's senders hold at least
                                   m * value / 1024 edges (0 = every superstep, 1025 = never; default 256) */
#define PGX_OPT_SEG_PREDICT 6   /* CC: the apply builds no frontier when the next superstep is
                                   predicted segmented, which then runs segmented (0 never,
                                   1 predicted -- default, 2 after every segmented superstep) */
#define PGX_OPT_PULL_MIN_EDGES 7 /* unit-weight SSSP with an in-CSR (pgx_sssp_run_dir): bottom-up
                                   superstep when its senders hold at least m * value / 1024 edges
                                   (0 = every superstep after the first, 1025 = never; default 128) */
#define PGX_OPT_COUNT 8

/* PGX_OPT_LAYOUT values (LayoutMode, layout.py:31-33).  EXTERNALISED is the
 * default SoA (value[], mailbox[] apart).  INTERLEAVED keeps one {mailbox,
 * value} record per vertex (the reference's AoS record, layout.py:85-129)
 * inside the run workspace; pgx_run_workspace_bytes sizes it, so set the
 * option before querying the size. */
#define PGX_LAYOUT_EXTERNALISED 0
#define PGX_LAYOUT_INTERLEAVED 1
int pgx_set_option(int key, int value);

/* number of SMs of `device` (host out pointer; syncs) */
int pgx_device_sm_count(int device, int *sm_count);

/* ---------------------------------------------------------------- */
/* graph preparation -- replaces the per-superstep work split of       */
/* scheduler.py:91-116 (edge_balanced_partition) with a one-time       */
/* edge-space tiling of the CSR                                        */
/* ---------------------------------------------------------------- */

/* int64 reference offsets (graph.py:28) -> int32 device row_ptr */
int pgx_offsets_to_i32(const int64_t *offsets64, int32_t *row_ptr,
                       int64_t count, uintptr_t stream);

/* bytes of the per-graph workspace for n vertices / m edges (host out) */
int pgx_graph_workspace_bytes(int64_t n, int64_t m, size_t *bytes);

/* build the compacted non-zero-degree source list and its edge tiles */
int pgx_graph_prepare(int32_t n, int64_t m, const int32_t *row_ptr,
                      void *graph_ws, size_t graph_ws_bytes,
                      uintptr_t stream);

/* ---------------------------------------------------------------- */
/* destination-segmented index (the dense supersteps' edge order) --   */
/* graph preparation for the segmented scatter of pgx_cc_run_ex /      */
/* pgx_sssp_run_ex, which combines every message of a dense superstep  */
/* in a shared-memory copy of its recipient's mailbox segment (the     */
/* paper's hybrid combiner, mailbox.py:180-199, for all recipients).   */
/* The edges are regrouped by destination segment (2^seg_log2          */
/* consecutive ids), CSR order kept inside a segment; an ENTRY is one  */
/* source's run of edges into one segment.                             */
/* ---------------------------------------------------------------- */

typedef struct PgxSegIndex {
  int32_t seg_log2;         /* segment = vertex >> seg_log2 (5..15)        */
  int32_t nent;             /* entries                                     */
  int32_t nitems;           /* work items                                  */
  int32_t reserved;
  const int32_t *ent_src;   /* [nent+4] source of each entry (16-byte
                               aligned; 4 slots of padding)                */
  const int32_t *ent_eb;    /* [nent+1] first edge (segment order); [nent] = m
                               (build output; the scatter finds entries from
                               col16's flags and does not read it: may be
                               NULL / freed for a run)                     */
  const uint16_t *col16;    /* [m+256]  shared-memory slot of (destination -
                               segment base), bank-swizzled; bit 15 flags
                               the first edge of an entry                  */
  const int32_t *tile_ent;  /* [ceil(m/256)+1] entry holding edge 256 t    */
  const int32_t *items;     /* [nitems][4] {segment, e0, e1, owns segment},
                               16-byte aligned, largest first              */
} PgxSegIndex;

/* default segment size (16384 vertices: a 64 KB shared-memory mailbox) */
#define PGX_SEG_LOG2_DEFAULT 14

/* workspace bytes of pgx_seg_count / pgx_seg_build (nent < 0: the count
 * step only) and the capacity the items array needs (host outs) */
int pgx_seg_workspace_bytes(int32_t n, int64_t m, int64_t nent,
                            int32_t seg_log2, size_t *bytes);
int pgx_seg_max_items(int32_t n, int64_t m, int32_t seg_log2,
                      int32_t *max_items);

/* Rectangular form (the partitioned path): nrows source rows, destinations
 * < ndst (pgx_seg_workspace_bytes / pgx_seg_max_items then take ndst). */
int pgx_seg_count_ex(int32_t nrows, int32_t ndst, int64_t m,
                     const int32_t *row_ptr, const int32_t *col_idx,
                     const void *graph_ws, int32_t seg_log2, void *ws,
                     size_t ws_bytes, int64_t *nent, uintptr_t stream);
int pgx_seg_build_ex(int32_t nrows, int32_t ndst, int64_t m,
                     const int32_t *row_ptr, const int32_t *col_idx,
                     const void *graph_ws, int32_t seg_log2, int64_t nent,
                     void *ws, size_t ws_bytes, int32_t *ent_src,
                     int32_t *ent_eb, uint16_t *col16, int32_t *tile_ent,
                     int32_t *items, int32_t *nitems, int32_t ctas,
                     uintptr_t stream);

/* step 1 (syncs): the number of entries into *nent (host out).  graph_ws
 * is the pgx_graph_prepare workspace of (row_ptr, col_idx). */
int pgx_seg_count(int32_t n, int64_t m, const int32_t *row_ptr,
                  const int32_t *col_idx, const void *graph_ws,
                  int32_t seg_log2, void *ws, size_t ws_bytes,
                  int64_t *nent, uintptr_t stream);

/* step 2 (syncs): fill the caller's arrays (sizes as in PgxSegIndex;
 * items: pgx_seg_max_items x 4 int32) and *nitems (host out).  Items are
 * cut for `ctas` persistent CTAs (0: the run kernels' grid). */
int pgx_seg_build(int32_t n, int64_t m, const int32_t *row_ptr,
                  const int32_t *col_idx, const void *graph_ws,
                  int32_t seg_log2, int64_t nent, void *ws, size_t ws_bytes,
                  int32_t *ent_src, int32_t *ent_eb, uint16_t *col16,
                  int32_t *tile_ent, int32_t *items, int32_t *nitems,
                  int32_t ctas, uintptr_t stream);

/* ---------------------------------------------------------------- */
/* whole runs on one GPU: one persistent cooperative kernel per run,   */
/* every superstep and the halt test on the device.                    */
/* Replaces _Executor.run (engine.py:255-316) for the lowered programs */
/* ---------------------------------------------------------------- */

/* bytes of the per-run workspace (host out) */
int pgx_run_workspace_bytes(int app, int64_t n, int64_t m,
                            int32_t max_supersteps, size_t *bytes);

/* Hub recipients (the paper's hybrid combiner split by recipient class):
 * optionally, col_idx may be an ENCODED copy in which every edge into one
 * of `nhubs` hub vertices holds (0x80000000 | slot), hub_ids[slot] being
 * the vertex; those edges are read-filtered and pre-combined in a per-CTA
 * shared-memory copy of the hub mailboxes.  nhubs = 0: plain col_idx.
 * nhubs <= pgx_hub_capacity(). */
int pgx_hub_capacity(int32_t *capacity);

/* sssp(source) -- algorithms.py:116-152 (push, min, uint32 hops) */
int pgx_sssp_run(int32_t n, int64_t m, const int32_t *row_ptr,
                 const int32_t *col_idx, const void *graph_ws,
                 const int32_t *hub_ids, int32_t nhubs,
                 int32_t source, int32_t max_supersteps, uint32_t *dist,
                 void *run_ws, size_t run_ws_bytes, int64_t *stats,
                 uintptr_t stream);

/* connected_components() -- algorithms.py:87-113 (Hashmin, min) */
int pgx_cc_run(int32_t n, int64_t m, const int32_t *row_ptr,
               const int32_t *col_idx, const void *graph_ws,
               const int32_t *hub_ids, int32_t nhubs,
               int32_t max_supersteps, uint32_t *labels, void *run_ws,
               size_t run_ws_bytes, int64_t *stats, uintptr_t stream);

/* the same runs with a segmented index (NULL: K1 for every superstep):
 * supersteps whose senders hold enough edges (PGX_OPT_SEG_MIN_EDGES) run
 * the segmented shared-memory scatter.  Results and statistics are
 * identical; the index must describe (row_ptr, col_idx). */
int pgx_sssp_run_ex(int32_t n, int64_t m, const int32_t *row_ptr,
                    const int32_t *col_idx, const void *graph_ws,
                    const PgxSegIndex *seg, int32_t source,
                    int32_t max_supersteps, uint32_t *dist, void *run_ws,
                    size_t run_ws_bytes, int64_t *stats, uintptr_t stream);
/* unit-weight SSSP, direction-optimising: as pgx_sssp_run_ex (seg may be
 * NULL), plus the in-CSR (in_row_ptr / in_col: the transpose of (row_ptr,
 * col_idx), rows sorted by source id).  A superstep whose senders hold at
 * least PGX_OPT_PULL_MIN_EDGES of the edges runs bottom-up: every vertex
 * tests its in-edges against the senders bitmap until the first sender
 * (the has-message bitmask is the superstep's whole result, every message
 * of a superstep being equal).  Results and statistics are identical to
 * pgx_sssp_run. */
int pgx_sssp_run_dir(int32_t n, int64_t m, const int32_t *row_ptr,
                     const int32_t *col_idx, const void *graph_ws,
                     const PgxSegIndex *seg, const int32_t *in_row_ptr,
                     const int32_t *in_col, int32_t source,
                     int32_t max_supersteps, uint32_t *dist, void *run_ws,
                     size_t run_ws_bytes, int64_t *stats, uintptr_t stream);
int pgx_cc_run_ex(int32_t n, int64_t m, const int32_t *row_ptr,
                  const int32_t *col_idx, const void *graph_ws,
                  const PgxSegIndex *seg, int32_t max_supersteps,
                  uint32_t *labels, void *run_ws, size_t run_ws_bytes,
                  int64_t *stats, uintptr_t stream);

/* pagerank(iterations, damping) -- algorithms.py:27-84 (fp64, sum).
 * base = (1 - damping) / n and r0 = 1 / n are passed in as computed by
 * the host (Python float arithmetic, algorithms.py:49-50). */
int pgx_pagerank_run(int32_t n, int64_t m, const int32_t *row_ptr,
                     const int32_t *col_idx, const void *graph_ws,
                     int32_t iterations, double damping, double base,
                     double r0, int32_t max_supersteps, double *rank,
                     void *run_ws, size_t run_ws_bytes, int64_t *stats,
                     uintptr_t stream);

/* pagerank(iterations, damping) in pull mode -- the reference's own comm
 * mode for PR (algorithms.py:80; fold engine.py:425-457): every vertex
 * folds its in-neighbours' shares, no atomics.  Needs the in-CSR
 * (in_row_ptr / in_col, rows sorted by source id) and its graph workspace
 * from pgx_graph_prepare(in_row_ptr); row_ptr gives the out-degrees.
 * in_col must be 32-byte aligned (256-bit id loads); every other array
 * needs only its element alignment. */
int pgx_pagerank_pull_run(int32_t n, int64_t m, const int32_t *row_ptr,
                          const int32_t *in_row_ptr, const int32_t *in_col,
                          const void *in_graph_ws, int32_t iterations,
                          double damping, double base, double r0,
                          int32_t max_supersteps, double *rank, void *run_ws,
                          size_t run_ws_bytes, int64_t *stats,
                          uintptr_t stream);

/* connected_components() from host memory with superstep 0 hidden under the
 * upload (engine.py:255-316's first superstep: every vertex sends its id).
 * pgx_cc_prescatter_init clears the run's mailbox / has-bitmask; once the
 * offsets and the tile map (pgx_graph_prepare) are on the device,
 * pgx_cc_source_scatter combines the messages of the edges [e_lo, e_hi)
 * (only those targets need to have landed) -- call it for every chunk as
 * its copy completes, on one stream; pgx_cc_run_prescattered then runs
 * the remaining supersteps (K1, shipped options) from the apply of
 * superstep 0.  Same labels and statistics as pgx_cc_run. */
int pgx_cc_prescatter_init(int32_t n, int64_t m, int32_t max_supersteps, void *run_ws,
                           size_t run_ws_bytes, uintptr_t stream);
int pgx_cc_source_scatter(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
                          const void *graph_ws, int64_t e_lo, int64_t e_hi,
                          int32_t max_supersteps, void *run_ws, size_t run_ws_bytes,
                          uintptr_t stream);
int pgx_cc_run_prescattered(int32_t n, int64_t m, const int32_t *row_ptr,
                            const int32_t *col_idx, const void *graph_ws,
                            int32_t max_supersteps, uint32_t *labels, void *run_ws,
                            size_t run_ws_bytes, int64_t *stats, uintptr_t stream);

/* Hub sources of the pull fold (the north star's hybrid path, pull form):
 * in_col_hubs is a copy of in_col in which every edge FROM one of `nhubs`
 * hub sources (the highest out-degree vertices) holds (0x80000000 | slot);
 * hub_slot[v] is v's slot or -1 (n entries).  Each CTA keeps the hub
 * shares in shared memory, so those edges cost no scattered global load.
 * Results are bit-identical to pgx_pagerank_pull_run.  Replaces the same
 * reference interface (engine.py:425-457 fold, algorithms.py:27-84).
 * nhubs <= pgx_pr_hub_capacity(); nhubs = 0 is pgx_pagerank_pull_run. */
int pgx_pr_hub_capacity(int32_t *capacity);
int pgx_pagerank_pull_hubs_run(int32_t n, int64_t m, const int32_t *row_ptr,
                               const int32_t *in_row_ptr, const int32_t *in_col_hubs,
                               const void *in_graph_ws, const int32_t *hub_slot,
                               int32_t nhubs, int32_t iterations, double damping,
                               double base, double r0, int32_t max_supersteps,
                               double *rank, void *run_ws, size_t run_ws_bytes,
                               int64_t *stats, uintptr_t stream);

/* ---------------------------------------------------------------- */
/* phases of the partitioned multi-GPU superstep.     */
/* A rank owns the out-edges of vertices [lo, lo+len) (a local CSR     */
/* with GLOBAL destination ids) and that slice of the mailbox.  Per    */
/* superstep the host calls pgx_scatter (into a full-width local       */
/* mailbox), reduces the slices onto their owners (NCCL min / sum via  */
/* torch.distributed), then pgx_apply_slice / pgx_pr_apply_slice --    */
/* or, for min programs, pgx_scatter_peer, which combines straight     */
/* into the owners' mailboxes over peer memory (no reduction).         */
/* Replaces the same reference functions as the *_run entry points,    */
/* one phase at a time.                                                */
/* ---------------------------------------------------------------- */

/* value / rank / share initialisation of an owned slice (setup,
 * algorithms.py:44-59, 96-97, 129-134); `val` is u32 labels/distances or
 * f64 ranks; `share`/`row_ptr` for PageRank only */
int pgx_slice_init(int app, int32_t len, int32_t lo, void *val,
                   const int32_t *row_ptr, double *share, double r0,
                   uintptr_t stream);

/* K1 alone: senders push along out-edges into `mailbox` (global ids).
 * dense != 0: senders are a graph workspace's non-zero-degree list
 * (src_eb = its row starts, src_ids = its local ids; min: message =
 * id + id_offset; sum: message = ((double*)src_msg)[id]);
 * dense == 0: a frontier built by pgx_apply_slice (src_eb/src_rs/src_msg).
 * has_bits may be NULL. */
int pgx_scatter(int op, int dense, const int32_t *col_idx,
                const int32_t *src_eb, const int32_t *src_rs,
                const int32_t *src_ids, int32_t id_offset, const void *src_msg,
                const int32_t *tile_src, int32_t nsrc, int64_t edges,
                void *mailbox, uint32_t *has_bits, uint32_t neutral,
                uintptr_t stream);

/* Sparse exchange, min programs.  The touched slots of
 * a full-width local mailbox are its set has-bits; pgx_touched counts those
 * outside [lo, hi) into *count (device int64) and, when `pairs` is not
 * NULL, compacts them in vertex order (hence grouped by owner) into
 * (slot << 32 | value) pairs, resetting each compacted slot to `neutral`.
 * scratch: pgx_touched_scratch_bytes(n).  pgx_scatter_pairs min-combines
 * received pairs into a mailbox (global slot ids). */
int pgx_touched_scratch_bytes(int32_t n, size_t *bytes);
int pgx_touched(int32_t n, int32_t lo, int32_t hi, const uint32_t *has_bits,
                uint32_t *mailbox, uint32_t neutral, uint64_t *pairs,
                int64_t *count, void *scratch, uintptr_t stream);
int pgx_scatter_pairs(const uint64_t *pairs, int64_t count, uint32_t *mailbox,
                      uintptr_t stream);

/* Fused peer-memory exchange (min programs): the compute step and the
 * collective in ONE kernel.  Like pgx_scatter(PGX_OP_MIN_U32, ...) into this
 * rank's full-width `mailbox` (its local filter), and every message that
 * passes the filter with a recipient outside [lo, hi) is also combined with
 * a fire-and-forget red.min into the owner's slot, peer_mailboxes[owner] +
 * v (device array of `world` base pointers: NVLink peer mappings from
 * pgx_peer_open, or this process's own pointers); owners come from the
 * device array bounds[world + 1].  The kernel ends with a system-scope
 * fence, so the collective the caller issues after it on the stream (the
 * counters all-reduce) orders every peer combine before the owners' apply.
 * No mailbox reduction is needed afterwards.  Replaces send_hybrid /
 * apply_cas (mailbox.py:147-199) across GPUs. */
int pgx_scatter_peer(int dense, const int32_t *col_idx, const int32_t *src_eb,
                     const int32_t *src_rs, const int32_t *src_ids,
                     int32_t id_offset, const void *src_msg,
                     const int32_t *tile_src, int32_t nsrc, int64_t edges,
                     uint32_t *mailbox, uint32_t *has_bits, uint32_t neutral,
                     const uint64_t *peer_mailboxes, const int32_t *bounds,
                     int32_t world, int32_t lo, int32_t hi, uintptr_t stream);

/* After a peer-exchange superstep: reset the foreign slots this rank
 * touched (set has-bits outside [lo, hi)) to `neutral`, clear every
 * has-bit.  Owned slots are consumed by pgx_apply_slice. */
int pgx_reset_touched(int32_t n, int32_t lo, int32_t hi, uint32_t *has_bits,
                      uint32_t *mailbox, uint32_t neutral, uintptr_t stream);

/* Unit-weight SSSP over the peer exchange, as bitmaps (the partitioned form
 * of the single-GPU has-bitmap filter): every message of a superstep is the
 * same level, so a recipient needs only its has-bit.  pgx_scatter_peer_bfs:
 * K1 over the rank's frontier filtering on its own full-width has-bitmap
 * (the local filter copy); a clear bit is set locally and, when another
 * rank owns the recipient, also in that owner's has-bitmap with a
 * system-scope red.or over peer memory (peer_has[world] base pointers;
 * owned bits use system scope too).  lo/hi: the rank's owned range of
 * bitmap positions (whole 32-bit words).  pgx_apply_slice_bfs: the owned
 * block's set bits are the recipients (has_block = the owned words);
 * unreached ones take distance `level` and, with out-edges, join the next
 * frontier (message level + 1); the block's words are then cleared
 * (count_only: counted, left set). */
int pgx_scatter_peer_bfs(const int32_t *col_idx, const int32_t *src_eb,
                         const int32_t *src_rs, const void *src_msg,
                         const int32_t *tile_src, int32_t nsrc, int64_t edges,
                         uint32_t *has_bits, const uint64_t *peer_has,
                         const int32_t *bounds, int32_t world, int32_t lo,
                         int32_t hi, uintptr_t stream);
int pgx_apply_slice_bfs(int32_t len, const int32_t *row_ptr, uint32_t *dist,
                        uint32_t *has_block, int32_t *f_eb, int32_t *f_rs,
                        uint32_t *f_msg, int32_t *tile_src, void *counters,
                        int32_t count_only, uint32_t level, uintptr_t stream);

/* Mailboxes other processes can map (CUDA IPC over NVLink / NVSwitch):
 * pgx_peer_alloc = cudaMalloc + its IPC handle (PGX_IPC_HANDLE_BYTES,
 * may be NULL); pgx_peer_open maps another process's handle (peer access
 * enabled lazily); pgx_peer_close unmaps; pgx_peer_free frees. */
#define PGX_IPC_HANDLE_BYTES 64
int pgx_peer_alloc(size_t bytes, void **ptr, void *ipc_handle);
int pgx_peer_open(const void *ipc_handle, void **ptr);
int pgx_peer_close(void *ptr);
int pgx_peer_free(void *ptr);
/* ranks that are threads of one process on different GPUs map each
 * other's mailboxes directly: enable peer access to `peer_device` from the
 * current device (already enabled: success) */
int pgx_peer_enable(int32_t peer_device);

/* size of the device counter block used by pgx_apply_slice (host out) */
int pgx_slice_counters_bytes(size_t *bytes);

/* K2 on an owned slice (min programs): recipients are the slots that are
 * not `neutral` after the reduction; consume (reset to `neutral`), adopt,
 * build the next frontier (edge prefix + tile map) and count.  count_only:
 * cap reached, only count recipients.  The partitioned path uses
 * neutral = INT32_MAX so that a signed int32 MIN reduction (NCCL / gloo)
 * is exact: every message is < n <= 2^31 - 1. */
int pgx_apply_slice(int app, int32_t len, const int32_t *row_ptr,
                    uint32_t *val, uint32_t *mailbox_slice, int32_t *f_eb,
                    int32_t *f_rs, uint32_t *f_msg, int32_t *tile_src,
                    void *counters, int32_t count_only, uint32_t neutral,
                    uint32_t *send_values, uintptr_t stream);
/* send_values (CC, may be NULL): the label every new sender sends is also
 * stored at send_values[local v] -- the input of pgx_seg_scatter; the
 * caller fills it with UINT32_MAX (no message) before the apply. */

/* K1s on a rank's slice (the dense supersteps of the partitioned CC): the
 * destination-segmented scatter (pgx_seg.cuh) of the rank's local CSR,
 * whose destinations are padded mailbox positions < ndst, built with
 * pgx_seg_count_ex / pgx_seg_build_ex (nrows = the rank's rows).  msg 0:
 * every entry's source sends its global id (local id + id_offset, CC
 * superstep 0); msg 1: it sends send_values[local source] (UINT32_MAX =
 * no message).  Writes exactly what pgx_scatter(PGX_OP_MIN_U32, ...)
 * would: the min-combined mailbox (untouched owned slots stored as
 * `neutral`) and its has-bits.  item_ctr: one device word of scratch. */
int pgx_seg_scatter(int msg, const PgxSegIndex *seg, int64_t m, int32_t ndst,
                    int32_t id_offset, const uint32_t *send_values,
                    uint32_t *mailbox, uint32_t *has_bits, uint32_t neutral,
                    unsigned *item_ctr, uintptr_t stream);

/* PageRank apply on an owned slice: rank, next share, per-CTA dangling
 * partials (partials[ceil(len/512)]).  `dangling` is a DEVICE scalar, the
 * job's dangling mass after the previous superstep (the all-reduce of
 * every rank's partials, issued on the stream: no host read); the kernel
 * uses dangling / n_total (algorithms.py:61-73). */
int pgx_pr_apply_slice(int32_t len, const int32_t *row_ptr, double *rank,
                       double *mailbox_slice, double *share, double base,
                       double damping, const double *dangling, double n_total,
                       int32_t last, double *partials, uintptr_t stream);

/* K3 on a rank's slice, the pull fold of the partitioned PageRank
 * (engine.py:425-457): in_col / in_graph_ws are the rank's local in-CSR
 * (rows = the nrows padded mailbox positions, entries = local source ids,
 * pgx_graph_prepare'd; nsrc = its non-zero row count, header word 0) and
 * `share` the rank's shares.  Writes the partial fold of every row that
 * lies inside one 256-edge tile into folded[row]; rows spanning tiles
 * leave tail / head partials ([ceil(m/256)+2] each) that
 * pgx_fold_spanning combines in tile order.  Rows without local in-edges
 * are not written (zero `folded` first).  No atomics; deterministic. */
int pgx_gather_slice(int32_t nrows, int64_t m, const int32_t *in_col,
                     const void *in_graph_ws, int32_t nsrc, const double *share,
                     double *folded, double *head, double *tail,
                     uintptr_t stream);
int pgx_fold_spanning(int32_t nspan, const int32_t *rows, const int32_t *t0,
                      const int32_t *t1, const double *head, const double *tail,
                      double *folded, uintptr_t stream);

/* ---------------------------------------------------------------- */
/* R-MAT input generator; input construction only.    */
/* Writes src << 32 | dst keys of the non-loop draws in                */
/* [first_draw, first_draw + num_draws) whose source lies in           */
/* [src_lo, src_hi) -- plus the reverse keys when `symmetric` -- into  */
/* keys[*count ...] (count is a device int64 counter, atomically       */
/* advanced; the caller sorts and dedups).                             */
/* ---------------------------------------------------------------- */
int pgx_rmat_keys(int32_t scale, int64_t first_draw, int64_t num_draws,
                  double a, double b, double c, uint64_t seed,
                  int32_t symmetric, int64_t src_lo, int64_t src_hi,
                  uint64_t *keys, int64_t capacity, int64_t *count,
                  uintptr_t stream);

/* ---------------------------------------------------------------- */
/* scattered-access ceilings (SURVEY.md 8(d) secondary roofline):      */
/* n_ops accesses of one kind to uniformly random slots of `buf`       */
/* (n_elems, a power of two), timed with CUDA events; host `ms` out,   */
/* syncs.                                                              */
/* ---------------------------------------------------------------- */
#define PGX_MB_LOAD_U32 0      /* read-filter: ld.global u32 */
#define PGX_MB_LOAD_F64 1      /* pull gather: ld.global.nc f64 */
#define PGX_MB_RED_MIN_U32 2   /* min combine: red.min.u32 */
#define PGX_MB_RED_ADD_F64 3   /* sum combine: red.add.f64 */
#define PGX_MB_ATOM_MIN_U32 4  /* atomicMin.u32 with return value */
#define PGX_MB_LOAD_U32_CG 5   /* ld.global.cg u32 (L2 only) */
#define PGX_MB_LOAD_U32_NA 6   /* ld.global.L1::no_allocate u32 */
#define PGX_MB_LOAD_U32_RELAXED 7  /* ld.relaxed.gpu u32 */
int pgx_microbench(int kind, void *buf, int64_t n_elems, int64_t n_ops,
                   uint64_t seed, float *ms, uintptr_t stream);

#ifdef __cplusplus
}
#endif

#endif /* PGX_H */
