// pgx_run.cu -- whole runs on one GPU: the persistent superstep kernels.
//
// One persistent cooperative kernel runs a whole Pregel run: every
// superstep's scatter (send + combine into the recipient mailbox), apply
// (consume + compute + vote-to-halt) and the halt test stay on the device,
// separated by a grid barrier.  Reference semantics:
//   engine.py:255-316   _Executor.run (BSP loop, stats, quiescence, cap)
//   engine.py:402-414   _chunk_push (consume, compute)
//   engine.py:154-162   send_to_out_neighbors (per-edge send)
//   mailbox.py:180-199  send_hybrid: publish-once + lock-free combine
//   mailbox.py:147-165  apply_cas: skip the atomic when combine is a no-op
//   algorithms.py       pagerank 27-84, connected_components 87-113,
//                       sssp 116-152
//   scheduler.py:91-116 edge_balanced_partition (edge-space split)
//
// Mapping of the paper's three optimisations onto sm_100a:
//   hybrid combiner  -> read-filter (plain load, skip when min(old,msg)==old)
//                       + one fire-and-forget red.min.u32 / red.add.f64;
//                       publication is an idempotent has-message bit set by
//                       every lane whose filter read saw the neutral
//                       (pgx_scatter.cuh).
//   externalisation  -> SoA: value[], mailbox[], has-bitmask, frontier SoA.
//   edge-centric     -> the frontier is built with its exclusive edge
//                       prefix (one 64-bit packed atomic per apply batch,
//                       pgx_apply.cuh); the scatter walks fixed 256-edge warp
//                       tiles of that edge space -- exact edge balance, hub
//                       rows split across tiles.
// Unit-weight SSSP filters on the has-message bitmap instead of the mailbox
// (every message of a superstep is equal; pgx_scatter.cuh, BFS = true).
// PageRank's default lowering is the reference's pull fold (pgx_gather.cuh).
#include "pgx_apply.cuh"
#include "pgx_common.cuh"
#include "pgx_gather.cuh"
#include "pgx_pull.cuh"
#include "pgx_scatter.cuh"
#include "pgx_seg.cuh"

// CC: the two send buffers are not initialised in the setup but cleared by
// the streaming stores under supersteps 0 and 1 (segmented, request-bound:
// the stores hide), 537 MB fewer setup writes on C5 (C2 -0.7 %, C5 -0.15 %)
#ifndef PGX_SV_LAZY
#define PGX_SV_LAZY 1
#endif

namespace pgx {
namespace {

// ------------------------------------------------------------------
// persistent run kernels
// ------------------------------------------------------------------

struct MinRunParams {
  int32_t n;
  int64_t m;
  const int32_t *row_ptr;
  const int32_t *col;
  GraphWs g;
  RunWs ws;
  uint32_t *val;
  int32_t source;  // SSSP only
  int32_t max_steps;
  int32_t read_filter;
  int32_t cas_loop;       // ablation arms (pgx_set_option)
  int32_t vertex_sched;
  int32_t interleaved;    // PGX_LAYOUT_INTERLEAVED: {mailbox, value} records in ws.mailbox
  const int32_t *hub_ids;
  int32_t nhubs;
  int64_t *stats;
  // segmented scatter (pgx_seg.cuh) for supersteps whose senders hold at
  // least seg_min_edges edges; use_seg = 0: K1 only
  PgxSegIndex seg;
  int32_t use_seg;
  int64_t seg_min_edges;
  int32_t seg_predict;  // PGX_OPT_SEG_PREDICT
  // bottom-up supersteps of unit-weight SSSP (pgx_pull.cuh) for supersteps
  // whose senders hold at least pull_min_edges edges; use_pull = 0: none
  const int32_t *in_row_ptr;
  const int32_t *in_col;
  int32_t use_pull;
  int64_t pull_min_edges;
};

// S = 0: externalised SoA (value = the caller's output array); S = 1:
// interleaved {mailbox, value} records (layout.py's INTERLEAVED), values
// copied out to the caller's array at the end of the run.
// ARMS = false: the shipped configuration (read-filter on, fire-and-forget
// combines, edge-balanced tiles, no hub cache) with the ablation arms
// compiled out, so they cost the hot loops no registers -- used for the
// unit-weight SSSP kernel (C3 -7 %); the CC kernel measured 1 % slower
// without them (code generation), so it keeps them
// PRE = true (CC, K1 only): superstep 0's messages are already in the
// mailbox / has-bitmask, scattered chunk by chunk while the CSR was being
// uploaded (pgx_cc_source_scatter); the kernel starts with the apply of
// superstep 0.  PRE = false compiles to the unchanged kernel.
template <int APP, int S, bool BFS = false, bool ARMS = true, bool PRE = false>
__global__ void __launch_bounds__(kBlock, PGX_MIN_BLOCKS) min_run_kernel(MinRunParams p) {
  extern __shared__ __align__(16) char smem[];
  __shared__ unsigned s_red[32];
  unsigned gen = 0;
  if (threadIdx.x == 0) gen = ld_acquire(&p.ws.bar->gen);
  uint32_t *mailbox = reinterpret_cast<uint32_t *>(p.ws.mailbox);
  uint32_t *val = S ? mailbox + 1 : p.val;
  const unsigned nthreads = gridDim.x * blockDim.x;
  const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;

  // ---- setup (algorithms.py:96-97 / 129-134) + superstep-0 senders ----
  // unit-weight SSSP on the shipped arm: the has-bit filter (scatter_phase);
  // the host launches the BFS instantiation only for the default options
  constexpr bool bfs = BFS && APP == PGX_APP_SSSP && S == 0;
  // send values (the segmented scatter's messages): CC labels; for
  // unit-weight SSSP any non-neutral value marks a sender (its messages are
  // uniform: the has-bitmask is the result)
  const bool use_sv = (APP == PGX_APP_CC || bfs) && p.use_seg;
#ifndef PGX_VAL_LAZY
#define PGX_VAL_LAZY 1
#endif
  // CC with the segmented scatter (PGX_VAL_LAZY): the labels are written by
  // streaming stores under superstep 0 (segmented: request-bound, the
  // stores hide), which does not read them
  const bool val_lazy = PGX_VAL_LAZY && APP == PGX_APP_CC && S == 0 && p.use_seg;
  for (unsigned v = gtid; v < (unsigned)p.n; v += nthreads) {
    if (!val_lazy) *slot<S>(val, v) = (APP == PGX_APP_CC) ? v : kNeutralMin;
    if (!BFS && !PRE) *slot<S>(mailbox, v) = kNeutralMin;  // the bitmap kernel has no mailbox
    // CC (PGX_SV_LAZY): the send buffers are cleared by the streaming
    // stores under the first two segmented supersteps instead (below)
    if (use_sv && !(PGX_SV_LAZY && APP == PGX_APP_CC)) p.ws.sv[0][v] = p.ws.sv[1][v] = kNeutralMin;
  }
  for (unsigned wi = gtid; wi < (unsigned)(p.n / 32 + 2); wi += nthreads) {
    if (!PRE) p.ws.has[wi] = 0u;
    p.ws.snd[0][wi] = 0u;
    p.ws.snd[1][wi] = 0u;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.stats[0] = p.stats[1] = 0;
    p.stats[2] = gridDim.x;
    p.stats[3] = (int64_t)globaltimer();
    StepCounters z = {};
    p.ws.ctr[0] = z;
    p.ws.ctr[1] = z;
    if (APP == PGX_APP_SSSP) {
      const int rs = p.row_ptr[p.source];
      const int deg = p.row_ptr[p.source + 1] - rs;
      if (deg > 0) {
        p.ws.f_eb[0] = 0;
        p.ws.f_rs[0] = rs;
        reinterpret_cast<uint32_t *>(p.ws.f_msg)[0] = 1u;
        for (int64_t t = 0; t * kTile < deg; t++) p.ws.tile_src[t] = 0;
        p.ws.ctr[0].packed = (1ull << 32) | (unsigned long long)deg;
      }
      p.ws.ctr[0].bcast = 1u;  // the source computes and sends in superstep 0
    } else {
      p.ws.ctr[0].bcast = (unsigned)p.n;  // every vertex broadcasts its id
    }
  }
  // the unit-weight SSSP kernel reads its per-superstep counters through
  // shared memory (grid_sync_bc); s_bc[0] = packed counts of the next
  // superstep's senders, s_bc[1] = recipients word, s_bc[2..3] scratch
  __shared__ unsigned long long s_bc[4];
// every min kernel reads its per-superstep counters through shared memory
// (C5 -0.15 %; with PGX_VAL_LAZY -0.3 %)
#ifndef PGX_BC_ALL
#define PGX_BC_ALL 1
#endif
  constexpr bool ctr_bc = bfs || PGX_BC_ALL;
  if constexpr (ctr_bc)
    grid_sync_bc(p.ws.bar, gen, &p.ws.ctr[0].packed, nullptr, s_bc);
  else
    grid_sync<kArriveRed>(p.ws.bar, gen);
  if (APP == PGX_APP_SSSP && gtid == 0) {
    *slot<S>(val, p.source) = 0u;
    if (p.row_ptr[p.source + 1] > p.row_ptr[p.source]) {  // the superstep-0 sender
      if (use_sv) p.ws.sv[0][p.source] = 1u;
      else p.ws.snd[0][p.source >> 5] = 1u << (p.source & 31);
    }
  }
  if (gtid == 0) p.stats[PGX_STAT_HDR + 7] = (int64_t)globaltimer();
  unsigned sv_stale = 0u;  // bit b: sv[b] may hold stale senders (grid-uniform)
  bool front_skipped = false;  // the last apply built no frontier (grid-uniform)
  int e_prev = (int)p.m;       // edges of the previous superstep (prediction)

  for (int s = 0;; s++) {
    // ---- scatter(s): senders push along out-edges into the mailbox ----
    const unsigned long long packed_s = ctr_bc ? s_bc[0] : p.ws.ctr[s].packed;
    const int64_t edges_s = (APP == PGX_APP_CC && s == 0) ? p.m
                                                          : (int64_t)(packed_s & 0xFFFFFFFFull);
    // a segmented superstep needs exact send values: after a K1 superstep
    // left them stale (below), K1 runs instead (never on C2 / C5, whose
    // dense supersteps come first)
    // (after an apply that predicted a segmented superstep and built no
    // frontier, the segmented pass runs whatever the edge count: a wrong
    // guess costs at most one dense pass; the send values are exact)
    // unit-weight SSSP: a superstep whose senders hold many edges runs
    // bottom-up (pgx_pull.cuh) -- the same has-bitmask from the receivers
    const bool pull_s = bfs && p.use_pull && s >= 1 && edges_s > 0 &&
                        edges_s >= p.pull_min_edges;
    const bool seg_s = !pull_s && p.use_seg && edges_s > 0 &&
                       (edges_s >= p.seg_min_edges || front_skipped) &&
                       !((sv_stale >> (s & 1)) & 1u);
    if (p.use_seg && ((PGX_SV_LAZY && APP == PGX_APP_CC && s <= 1) ||
                      (s >= 1 && (p.ws.ctr[s - 1].packed >> 32) != 0ull))) {
      // the send buffers of superstep s + 1, written by the next apply,
      // still hold the senders of s - 1 (last read by scatter(s - 1))
      if (use_sv) {
        // CC send values: cleared whole (a streaming store of n words)
        // under a segmented superstep, which hides it; otherwise the
        // buffer is marked stale and the superstep that would read it runs
        // K1 (never on C2 / C5, whose dense supersteps come first)
        if (seg_s) {
          uint4 *svx = reinterpret_cast<uint4 *>(p.ws.sv[(s + 1) & 1]);
          const uint4 nn = make_uint4(kNeutralMin, kNeutralMin, kNeutralMin, kNeutralMin);
          for (unsigned i = gtid; i < (unsigned)((p.n + 4) / 4); i += nthreads) svx[i] = nn;
          if (val_lazy && s == 0) {
            if ((reinterpret_cast<uintptr_t>(val) & 15u) == 0) {
              uint4 *vx = reinterpret_cast<uint4 *>(val);
              for (unsigned i = gtid; i < (unsigned)(p.n / 4); i += nthreads)
                vx[i] = make_uint4(4 * i, 4 * i + 1, 4 * i + 2, 4 * i + 3);
              for (unsigned v = (unsigned)(p.n & ~3) + gtid; v < (unsigned)p.n; v += nthreads) val[v] = v;
            } else {
              for (unsigned v = gtid; v < (unsigned)p.n; v += nthreads) val[v] = v;
            }
          }
          sv_stale &= ~(1u << ((s + 1) & 1));
        } else {
          sv_stale |= 1u << ((s + 1) & 1);
        }
      } else {
        // unit-weight SSSP senders bitmap: clear the set words
        uint32_t *nx = p.ws.snd[(s + 1) & 1];
        for (unsigned wi = gtid; wi < (unsigned)(p.n / 32 + 2); wi += nthreads)
          if (nx[wi]) nx[wi] = 0u;
      }
    }
    if (PRE && s == 0) {
      // superstep 0 was scattered during the upload (pgx_cc_source_scatter)
    } else if (pull_s) {
      if constexpr (bfs) {
        PullArgs pa;
        pa.in_row_ptr = p.in_row_ptr;
        pa.in_col = p.in_col;
        pa.dist = val;
        pa.n = p.n;
        pa.m = p.m;
        pa.level = (uint32_t)s;
        pa.snd = p.ws.snd[0];
        pa.has = p.ws.has;
        pa.q_eb = p.ws.f_eb;  // the frontier of superstep s is not read
        pa.q_rs = p.ws.f_rs;
        pa.q_v = reinterpret_cast<uint32_t *>(p.ws.f_msg);
        pa.q_tile = p.ws.tile_src;
        pa.q_ctr = p.ws.misc;
#ifndef PGX_PULL_TIMING
#define PGX_PULL_TIMING 0
#endif
        const uint64_t t0 = PGX_PULL_TIMING ? globaltimer() : 0;
        pull_senders_phase(pa);
        if (PGX_PULL_TIMING && gtid == 0) {
          p.ws.misc[2] = ~0ull;
          p.ws.misc[3] = 0ull;
          p.ws.misc[4] = ~0ull;
          p.ws.misc[5] = 0ull;
        }
        grid_sync<kArriveRed>(p.ws.bar, gen);
        const uint64_t t1 = PGX_PULL_TIMING ? globaltimer() : 0;
        pull_probe_phase(pa);
        if (PGX_PULL_TIMING) {  // debug build: spread of the CTAs' phase-B finish times
          __syncthreads();
          if (threadIdx.x == 0) {
            atomicMin(&p.ws.misc[2], (unsigned long long)globaltimer());
            atomicMax(&p.ws.misc[3], (unsigned long long)globaltimer());
          }
        }
        grid_sync_bc(p.ws.bar, gen, pa.q_ctr, nullptr, s_bc + 2);
        const uint64_t t2 = PGX_PULL_TIMING ? globaltimer() : 0;
        pull_remainder_phase(pa, s_bc[2], smem);
        if (PGX_PULL_TIMING) {  // debug build (tools): phase times of the pull superstep
          __syncthreads();
          if (threadIdx.x == 0) {
            atomicMin(&p.ws.misc[4], (unsigned long long)globaltimer());
            atomicMax(&p.ws.misc[5], (unsigned long long)globaltimer());
          }
          grid_sync<kArriveRed>(p.ws.bar, gen);
          if (gtid == 0)
            printf("pull s=%d A=%.1f B=%.1f (first CTA done %.1f, last %.1f) C=%.1f us "
                   "(first CTA done %.1f, last %.1f), remainder %u entries %u edges\n", s,
                   (t1 - t0) * 1e-3, (t2 - t1) * 1e-3, (p.ws.misc[2] - t1) * 1e-3,
                   (p.ws.misc[3] - t1) * 1e-3, (globaltimer() - t2) * 1e-3,
                   ((long long)p.ws.misc[4] - (long long)t2) * 1e-3,
                   ((long long)p.ws.misc[5] - (long long)t2) * 1e-3,
                   (unsigned)(*pa.q_ctr >> 32), (unsigned)(*pa.q_ctr & 0xFFFFFFFFull));
        }
      }
    } else if (seg_s) {
      // dense superstep: the segmented shared-memory scatter (pgx_seg.cuh)
      SegPass sp;
      sp.ix = p.seg;
      sp.m = p.m;
      sp.n = p.n;
      sp.snd = p.ws.snd[s & 1];
      sp.sv = use_sv ? p.ws.sv[s & 1] : nullptr;
      sp.uniform = (uint32_t)s + 1u;
      sp.mailbox = mailbox;
      sp.has = p.ws.has;
      sp.item_ctr = reinterpret_cast<unsigned *>(&p.ws.ctr[s].pad[0]);
      sp.write_mailbox = !bfs;
      sp.id_offset = 0;
      sp.out_neutral = kNeutralMin;
      if (APP == PGX_APP_CC && s == 0)
        seg_scatter_phase<kSegSourceId>(sp, smem);
      else
        seg_scatter_phase<kSegLabel>(sp, smem);
    } else {
    ScatterArgs a;
    a.col = p.col;
    a.mailbox = mailbox;
    a.has = p.ws.has;
    a.id_offset = 0;
    a.hub_ids = ARMS ? p.hub_ids : nullptr;
    a.nhubs = ARMS ? p.nhubs : 0;
    a.cas_loop = ARMS ? p.cas_loop : 0;
    const bool read_filter = ARMS ? (p.read_filter != 0) : true;
    const bool vertex_sched = ARMS && p.vertex_sched;
    a.neutral = kNeutralMin;
    a.n = p.n;
    if (APP == PGX_APP_CC && s == 0) {
      a.eb = p.g.nz_eb;
      a.rs = nullptr;
      a.ids = p.g.nz_id;
      a.msg = nullptr;
      a.tile_src = p.g.tile_src;
      a.nsrc = p.g.hdr[0];
      a.E = p.m;
      if (vertex_sched)
        scatter_vertex_phase<MsgSrc::kSourceId, S>(a, read_filter);
      else
        scatter_phase<PGX_OP_MIN_U32, MsgSrc::kSourceId, S>(a, smem, read_filter);
    } else {
      const unsigned long long packed = ctr_bc ? packed_s : p.ws.ctr[s].packed;
      a.eb = p.ws.f_eb;
      a.rs = p.ws.f_rs;
      a.ids = nullptr;
      a.msg = p.ws.f_msg;
      a.tile_src = p.ws.tile_src;
      a.nsrc = (int32_t)(packed >> 32);
      a.E = (int64_t)(packed & 0xFFFFFFFFull);
      if (vertex_sched)
        scatter_vertex_phase<MsgSrc::kFrontier, S>(a, read_filter);
      else if (bfs)
        scatter_phase<PGX_OP_MIN_U32, MsgSrc::kFrontier, 0, false, true>(a, smem);
      else
        scatter_phase<PGX_OP_MIN_U32, MsgSrc::kFrontier, S>(a, smem, read_filter);
    }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      StepCounters z = {};
      p.ws.ctr[s + 1] = z;
    }
    grid_sync<kArriveRed>(p.ws.bar, gen);
    const uint64_t t_scatter = globaltimer();

    // ---- apply(s+1): consume + compute + frontier build; at the cap the
    //      pending messages are only counted (engine.py:299-300) ----
    const bool at_cap = (s + 1 == p.max_steps);
    // senders bitmap for the unit-weight SSSP segmented pass; CC sends from
    // its send values alone
    uint32_t *snd_out = (p.use_seg && !use_sv) ? p.ws.snd[(s + 1) & 1] : nullptr;
    uint32_t *sv_out = use_sv ? p.ws.sv[(s + 1) & 1] : nullptr;
    // CC: predict whether superstep s+1 is segmented (it reads the send
    // values, not a frontier): this one is and the geometric edge trend
    // E_s * E_s / E_{s-1} stays above twice the threshold.  A wrong guess
    // runs the next superstep segmented anyway (at most one dense pass)
    const float e_s = (float)edges_s;
    const bool trend = e_s * (e_s / (float)max(e_prev, 1)) >= 2.0f * (float)p.seg_min_edges;
    const bool skip = use_sv && seg_s && !at_cap &&
                      (p.seg_predict == 2 || (p.seg_predict == 1 && trend));
    const unsigned long long rb =
        bfs ? apply_min_phase<APP, 0, true>(p.row_ptr, val, mailbox, p.n, p.ws, &p.ws.ctr[s + 1],
                                            smem, at_cap, (uint32_t)s + 1u, snd_out, sv_out, skip)
            : apply_min_phase<APP, S>(p.row_ptr, val, mailbox, p.n, p.ws, &p.ws.ctr[s + 1], smem,
                                      at_cap, 0u, snd_out, sv_out, skip);
    const unsigned bc = block_sum<unsigned>((unsigned)(rb & 0xFFFFFFFFull), s_red);
    const unsigned rc = block_sum<unsigned>((unsigned)(rb >> 32), s_red);
    if (threadIdx.x == 0) {
      if (bc) atomicAdd(&p.ws.ctr[s + 1].bcast, bc);
      if (rc) atomicAdd(&p.ws.ctr[s].recip, rc);
    }
    front_skipped = skip;
    e_prev = (int)edges_s;
    if constexpr (ctr_bc)
      grid_sync_bc(p.ws.bar, gen, &p.ws.ctr[s + 1].packed,
                   reinterpret_cast<const unsigned long long *>(&p.ws.ctr[s].recip), s_bc);
    else
      grid_sync<kArriveRed>(p.ws.bar, gen);

    // ---- stats + halt test (engine.py:284-300) ----
    const unsigned nrecip = ctr_bc ? (unsigned)s_bc[1] : p.ws.ctr[s].recip;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const StepCounters c = p.ws.ctr[s];
      const int64_t senders = (int64_t)(c.packed >> 32);
      const int64_t edges = (APP == PGX_APP_CC && s == 0) ? p.m : (int64_t)(c.packed & 0xFFFFFFFFull);
      const int64_t active = (s == 0) ? p.n : (int64_t)p.ws.ctr[s - 1].recip;
      const int64_t sent = (APP == PGX_APP_SSSP) ? edges : (int64_t)c.bcast;
      record_step(p.stats, s, active, sent, edges,
                  (APP == PGX_APP_CC && s == 0) ? (int64_t)p.g.hdr[0] : senders, nrecip,
                  (int64_t)c.bcast);
      p.stats[PGX_STAT_HDR + (int64_t)s * PGX_STAT_FIELDS + 5] = (int64_t)t_scatter;
      // scatter(s+1) starts after this barrier: field 7 of step s+1
      if (!at_cap)
        p.stats[PGX_STAT_HDR + (int64_t)(s + 1) * PGX_STAT_FIELDS + 7] = (int64_t)globaltimer();
      if (nrecip == 0) {
        p.stats[0] = s + 1;
      } else if (at_cap) {
        p.stats[0] = s + 1;
        p.stats[1] = 1;
      }
    }
    if (nrecip == 0 || at_cap) break;
  }
  if (S) {  // RunReport.values from the records (engine.py:310-311)
    for (unsigned v = gtid; v < (unsigned)p.n; v += nthreads) p.val[v] = *slot<S>(val, v);
  }
}

struct PrRunParams {
  int32_t n;
  int64_t m;
  const int32_t *row_ptr;
  const int32_t *col;
  GraphWs g;
  RunWs ws;
  double *rank;
  int32_t iterations;
  double damping, base, r0;
  int32_t max_steps;
  int64_t *stats;
};

__global__ void __launch_bounds__(kBlock, PGX_MIN_BLOCKS) pagerank_run_kernel(PrRunParams p) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double s_red[32];
  __shared__ unsigned long long s_ured[32];
  __shared__ double s_dangling;
  unsigned gen = 0;
  if (threadIdx.x == 0) gen = ld_acquire(&p.ws.bar->gen);
  double *mailbox = reinterpret_cast<double *>(p.ws.mailbox);
  double *share = reinterpret_cast<double *>(p.ws.f_msg);
  const unsigned nthreads = gridDim.x * blockDim.x;
  const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int last = p.iterations - 1;
  const double dn_n = (double)p.n;

  // ---- setup (algorithms.py:44-59): rank = r0, seed shares r0/outdeg ----
  unsigned long long my_dangling = 0;
  for (unsigned v = gtid; v < (unsigned)p.n; v += nthreads) {
    const int deg = p.row_ptr[v + 1] - p.row_ptr[v];
    p.rank[v] = p.r0;
    mailbox[v] = 0.0;
    share[v] = deg ? __ddiv_rn(p.r0, (double)deg) : 0.0;
    my_dangling += deg ? 0ull : 1ull;
  }
  unsigned long long bd = block_sum<unsigned long long>(my_dangling, s_ured);
  if (threadIdx.x == 0) {
    if (bd) atomicAdd(&p.ws.misc[0], bd);
    if (blockIdx.x == 0) {
      p.stats[0] = p.stats[1] = 0;
      p.stats[2] = gridDim.x;
      p.stats[3] = (int64_t)globaltimer();
    }
  }
  grid_sync(p.ws.bar, gen);

  ScatterArgs a;
  a.col = p.col;
  a.eb = p.g.nz_eb;
  a.rs = nullptr;
  a.ids = p.g.nz_id;
  a.msg = share;
  a.tile_src = p.g.tile_src;
  a.nsrc = p.g.hdr[0];
  a.E = p.m;
  a.mailbox = mailbox;
  a.has = nullptr;
  a.id_offset = 0;
  a.hub_ids = nullptr;
  a.nhubs = 0;
  a.cas_loop = 0;
  a.neutral = 0u;
  a.n = p.n;
  const unsigned long long ndangling = p.ws.misc[0];
  double dangling = __dmul_rn(p.r0, (double)ndangling);  // algorithms.py:55
  const int64_t nspread = (int64_t)p.n - (int64_t)ndangling;

  // the setup seed is folded in superstep 0 (algorithms.py:56-59)
  scatter_phase<PGX_OP_SUM_F64, MsgSrc::kShareById>(a, smem);
  grid_sync(p.ws.bar, gen);

  for (int s = 0;; s++) {
    // ---- apply(s): rank = base + d * (folded + dangling / n) ----
    const double dn = __ddiv_rn(dangling, dn_n);
    double my_d = 0.0;
    for (unsigned v = gtid; v < (unsigned)p.n; v += nthreads) {
      const double folded = mailbox[v];
      mailbox[v] = 0.0;
      const double r = __dadd_rn(p.base, __dmul_rn(p.damping, __dadd_rn(folded, dn)));
      p.rank[v] = r;
      const int deg = p.row_ptr[v + 1] - p.row_ptr[v];
      if (deg == 0) my_d = __dadd_rn(my_d, r);
      else if (s != last) share[v] = __ddiv_rn(r, (double)deg);
    }
    const double bsum = block_sum<double>(my_d, s_red);
    if (threadIdx.x == 0) p.ws.partials[blockIdx.x] = bsum;
    grid_sync(p.ws.bar, gen);

    // ---- on_superstep_end (algorithms.py:75-78): dangling mass ----
    {
      double acc = 0.0;
      for (int b = threadIdx.x; b < (int)gridDim.x; b += kBlock) acc = __dadd_rn(acc, p.ws.partials[b]);
      const double tot = block_sum<double>(acc, s_red);
      if (threadIdx.x == 0) s_dangling = tot;
      __syncthreads();
      dangling = s_dangling;
    }
    const bool cap = (s + 1 == p.max_steps);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      p.stats[PGX_STAT_HDR + (int64_t)s * PGX_STAT_FIELDS + 7] = (int64_t)globaltimer();
      record_step(p.stats, s, p.n, (s == last) ? 0 : nspread, p.m, nspread, p.n,
                  (s == last) ? 0 : nspread);
      if (s == last || cap) {
        p.stats[0] = s + 1;
        p.stats[1] = (s == last) ? 0 : 1;
      }
    }
    if (s == last || cap) break;
    scatter_phase<PGX_OP_SUM_F64, MsgSrc::kShareById>(a, smem);
    grid_sync(p.ws.bar, gen);
  }
}

#ifndef PGX_SSSP_BFS
#define PGX_SSSP_BFS 1
#endif
#ifndef PGX_PR_UNROLL
#define PGX_PR_UNROLL 2
#endif
constexpr int kPrUnroll = PGX_PR_UNROLL;

struct PrPullParams {
  int32_t n;
  int64_t m;
  const int32_t *row_ptr;     // out-CSR offsets (out-degrees)
  const int32_t *in_row_ptr;  // in-CSR offsets
  const int32_t *in_col;
  GraphWs gin;                // tile map / nz list of the in-CSR
  RunWs ws;
  double *rank;
  int32_t iterations;
  double damping, base, r0;
  int32_t max_steps;
  int64_t *stats;
  const int32_t *hub_slot;    // HUBS: [n] slot of a hub source, -1 otherwise
  int32_t nhubs;
};

// HUBS: the in-CSR holds (0x80000000 | slot) for edges from the nhubs hub
// sources; the compute writes their next shares to a compact slot-indexed
// array as well, and every CTA copies it into shared memory (coalesced)
// before each fold (pgx_gather.cuh)
template <bool HUBS>
__global__ void __launch_bounds__(kBlock, PGX_MIN_BLOCKS) pagerank_pull_kernel(PrPullParams p) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double s_red[32];
  __shared__ unsigned long long s_ured[32];
  __shared__ double s_dangling;
  unsigned gen = 0;
  double *folded = reinterpret_cast<double *>(p.ws.mailbox);
  double *share_cur = reinterpret_cast<double *>(p.ws.f_msg);
  double *share_nxt = p.ws.share2;
  double *hub_cur = p.ws.hub_share[0];
  double *hub_nxt = p.ws.hub_share[1];
  double *s_hub = reinterpret_cast<double *>(smem + (size_t)kWarps * kSlots * 8);
  const unsigned nthreads = gridDim.x * blockDim.x;
  const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int last = p.iterations - 1;
  const double dn_n = (double)p.n;

  // ---- setup (algorithms.py:44-59): rank = r0, seed shares r0/outdeg ----
  unsigned long long my_dangling = 0;
  for (unsigned v = gtid; v < (unsigned)p.n; v += nthreads) {
    const int deg = p.row_ptr[v + 1] - p.row_ptr[v];
    p.rank[v] = p.r0;
    const double sh = deg ? __ddiv_rn(p.r0, (double)deg) : 0.0;
    share_cur[v] = sh;
    if (HUBS) {
      const int slot = p.hub_slot[v];
      if (slot >= 0) hub_cur[slot] = sh;
    }
    my_dangling += deg ? 0ull : 1ull;
  }
  unsigned long long bd = block_sum<unsigned long long>(my_dangling, s_ured);
  if (threadIdx.x == 0) {
    if (bd) atomicAdd(&p.ws.misc[0], bd);
    if (blockIdx.x == 0) {
      p.stats[0] = p.stats[1] = 0;
      p.stats[2] = gridDim.x;
      p.stats[3] = (int64_t)globaltimer();
    }
  }
  grid_sync(p.ws.bar, gen);
  const unsigned long long ndangling = p.ws.misc[0];
  double dangling = __dmul_rn(p.r0, (double)ndangling);  // algorithms.py:55
  const int64_t nspread = (int64_t)p.n - (int64_t)ndangling;

  GatherArgs g;
  g.in_col = p.in_col;
  g.eb = p.gin.nz_eb;
  g.ids = p.gin.nz_id;
  g.tile_src = p.gin.tile_src;
  g.nsrc = p.gin.hdr[0];
  g.E = p.m;
  g.folded = folded;
  g.head = p.ws.head;
  g.tail = p.ws.tail;
  g.n = p.n;
  g.s_hub = s_hub;

  for (int s = 0;; s++) {
    if (blockIdx.x == 0 && threadIdx.x == 0)
      p.stats[PGX_STAT_HDR + (int64_t)s * PGX_STAT_FIELDS + 7] = (int64_t)globaltimer();
    if (HUBS) {  // the hub shares of last superstep into shared memory
      const double2 *src = reinterpret_cast<const double2 *>(hub_cur);
      double2 *dst = reinterpret_cast<double2 *>(s_hub);
      for (int h = threadIdx.x; h < (p.nhubs + 1) / 2; h += kBlock) dst[h] = __ldcg(src + h);
      __syncthreads();
    }
    // ---- fold (engine.py:425-457): in-neighbour shares of last superstep
    g.share = share_cur;
    gather_phase<HUBS>(g, smem);
    grid_sync(p.ws.bar, gen);
    const uint64_t t_fold = globaltimer();

    // ---- compute (algorithms.py:61-73): rank, next share, dangling mass
    // kPrUnroll vertices per thread and iteration, every load independent
    // (folded[v] is read unconditionally), so a thread keeps 5 * kPrUnroll
    // loads in flight instead of one dependent chain per vertex
    const double dn = __ddiv_rn(dangling, dn_n);
    double my_d = 0.0;
    for (unsigned v0 = gtid; v0 < (unsigned)p.n; v0 += kPrUnroll * nthreads) {
      int es[kPrUnroll], ee[kPrUnroll], r0[kPrUnroll], r1[kPrUnroll], hs[kPrUnroll];
      double fv[kPrUnroll];
#pragma unroll
      for (int j = 0; j < kPrUnroll; j++) {
        const unsigned v = v0 + j * nthreads;
        if (v < (unsigned)p.n) {
          es[j] = p.in_row_ptr[v];
          ee[j] = p.in_row_ptr[v + 1];
          r0[j] = p.row_ptr[v];
          r1[j] = p.row_ptr[v + 1];
          fv[j] = folded[v];
          if (HUBS) hs[j] = p.hub_slot[v];
        }
      }
#pragma unroll
      for (int j = 0; j < kPrUnroll; j++) {
        const unsigned v = v0 + j * nthreads;
        if (v >= (unsigned)p.n) continue;
        double f = 0.0;
        if (ee[j] > es[j]) {
          const int64_t t0 = es[j] / kTile, t1 = (ee[j] - 1) / kTile;
          if (t0 == t1) {
            f = fv[j];
          } else {
            f = span_sum(p.ws.head, p.ws.tail, t0, t1);
          }
        }
        const double r = __dadd_rn(p.base, __dmul_rn(p.damping, __dadd_rn(f, dn)));
        p.rank[v] = r;
        const int deg = r1[j] - r0[j];
        if (deg == 0) my_d = __dadd_rn(my_d, r);
        else if (s != last) {
          const double sh = __ddiv_rn(r, (double)deg);
          share_nxt[v] = sh;
          if (HUBS && hs[j] >= 0) hub_nxt[hs[j]] = sh;
        }
      }
    }
    const double bsum = block_sum<double>(my_d, s_red);
    if (threadIdx.x == 0) p.ws.partials[blockIdx.x] = bsum;
    grid_sync(p.ws.bar, gen);

    // ---- on_superstep_end (algorithms.py:75-78): dangling mass ----
    {
      double acc = 0.0;
      for (int b = threadIdx.x; b < (int)gridDim.x; b += kBlock) acc = __dadd_rn(acc, p.ws.partials[b]);
      const double tot = block_sum<double>(acc, s_red);
      if (threadIdx.x == 0) s_dangling = tot;
      __syncthreads();
      dangling = s_dangling;
    }
    const bool cap = (s + 1 == p.max_steps);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      record_step(p.stats, s, p.n, (s == last) ? 0 : nspread, p.m, nspread, p.n,
                  (s == last) ? 0 : nspread);
      p.stats[PGX_STAT_HDR + (int64_t)s * PGX_STAT_FIELDS + 5] = (int64_t)globaltimer();
#if PGX_PR_FOLD_STAMP  // timing probe builds: the fold's end in field 6
      p.stats[PGX_STAT_HDR + (int64_t)s * PGX_STAT_FIELDS + 6] = (int64_t)t_fold;
#endif
      (void)t_fold;
      if (s == last || cap) {
        p.stats[0] = s + 1;
        p.stats[1] = (s == last) ? 0 : 1;
      }
    }
    if (s == last || cap) break;
    double *tmp = share_cur;
    share_cur = share_nxt;
    share_nxt = tmp;
    tmp = hub_cur;
    hub_cur = hub_nxt;
    hub_nxt = tmp;
  }
}


inline size_t scatter_smem_bytes(int op) { return scatter_smem(op); }

}  // namespace
}  // namespace pgx

using namespace pgx;

extern "C" {

int pgx_run_workspace_bytes(int app, int64_t n, int64_t m, int32_t max_supersteps,
                            size_t *bytes) {
  if (!bytes || n < 0 || m < 0 || max_supersteps < 1 || app < 0 || app > 3)
    return fail(PGX_EINVAL, "bad run workspace arguments");
  *bytes = run_ws_layout(app, n, m, max_supersteps, nullptr, nullptr,
                         g_opt[PGX_OPT_LAYOUT] == PGX_LAYOUT_INTERLEAVED);
  return PGX_OK;
}

static int min_run(int app, int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
                   const void *graph_ws, const int32_t *hub_ids, int32_t nhubs,
                   int32_t source, int32_t max_supersteps, uint32_t *val,
                   void *run_ws, size_t run_ws_bytes, int64_t *stats, uintptr_t stream,
                   const PgxSegIndex *seg = nullptr, const int32_t *in_row_ptr = nullptr,
                   const int32_t *in_col = nullptr, bool pre = false) {
  if (nhubs < 0 || nhubs > kHubs || (nhubs > 0 && !hub_ids))
    return fail(PGX_EINVAL, "hub count must be in [0, pgx_hub_capacity()]");
  if (seg) {
    if (seg->seg_log2 < 5 || seg->seg_log2 > kSegMaxLog2 || seg->nent < 1 || seg->nent > m ||
        seg->nitems < 1 || !seg->ent_src || !seg->col16 || !seg->tile_ent ||
        !seg->items || reinterpret_cast<uintptr_t>(seg->items) % 16 ||
        reinterpret_cast<uintptr_t>(seg->ent_src) % 16 ||
        reinterpret_cast<uintptr_t>(seg->col16) % 16)
      return fail(PGX_EINVAL, "malformed segmented index");
  }
  if (g_opt[PGX_OPT_VERTEX_SCHED] && nhubs > 0)
    return fail(PGX_EINVAL, "the vertex-scheduled ablation arm has no hub cache");
  int rc = check_graph(n, m, row_ptr, col_idx, graph_ws);
  if (rc) return rc;
  if (max_supersteps < 1) return fail(PGX_EINVAL, "superstep cap must be >= 1");
  if (!val || !run_ws || !stats) return fail(PGX_EINVAL, "null output pointer");
  if (app == PGX_APP_SSSP && (source < 0 || source >= n))
    return fail(PGX_EINVAL, "source vertex out of range");
  MinRunParams p;
  p.n = n;
  p.m = m;
  p.row_ptr = row_ptr;
  p.col = col_idx;
  graph_ws_layout(n, m, &p.g, (char *)graph_ws);
  p.interleaved = g_opt[PGX_OPT_LAYOUT] == PGX_LAYOUT_INTERLEAVED;
  if (run_ws_layout(app, n, m, max_supersteps, &p.ws, (char *)run_ws, p.interleaved) >
      run_ws_bytes)
    return fail(PGX_ENOMEM, "run workspace too small");
  p.val = val;
  p.source = source;
  p.max_steps = max_supersteps;
  p.read_filter = g_opt[PGX_OPT_READ_FILTER];
  p.cas_loop = g_opt[PGX_OPT_CAS_LOOP];
  p.vertex_sched = g_opt[PGX_OPT_VERTEX_SCHED];
  p.hub_ids = hub_ids;
  p.nhubs = nhubs;
  p.stats = stats;
  cudaStream_t st = (cudaStream_t)stream;
  PGX_CUDA(cudaMemsetAsync(p.ws.bar, 0, 64, st));
  const bool shipped = p.read_filter && !p.cas_loop && !p.vertex_sched && nhubs == 0;
  const bool bfs = PGX_SSSP_BFS && !p.interleaved && shipped;
  // the segmented scatter runs on the shipped arm only (SoA, read-filter,
  // fire-and-forget combines, edge-balanced tiles, no hub cache)
  p.use_seg = seg && m > 0 && !p.interleaved && p.read_filter && !p.cas_loop && !p.vertex_sched &&
              nhubs == 0 && g_opt[PGX_OPT_SEG_MIN_EDGES] <= 1024;
  if (p.use_seg) p.seg = *seg;
  else memset(&p.seg, 0, sizeof p.seg);
  p.seg_min_edges = (m * (int64_t)g_opt[PGX_OPT_SEG_MIN_EDGES]) / 1024;
  p.seg_predict = g_opt[PGX_OPT_SEG_PREDICT];
  // bottom-up supersteps: the unit-weight (bitmap) kernel with an in-CSR
  p.in_row_ptr = in_row_ptr;
  p.in_col = in_col;
  p.use_pull = app == PGX_APP_SSSP && bfs && in_row_ptr && (m == 0 || in_col) &&
               g_opt[PGX_OPT_PULL_MIN_EDGES] <= 1024;
  p.pull_min_edges = (m * (int64_t)g_opt[PGX_OPT_PULL_MIN_EDGES]) / 1024;
  if (pre && (app != PGX_APP_CC || p.use_seg || p.interleaved || !shipped))
    return fail(PGX_EINVAL, "a pre-scattered run is CC on K1 with the shipped options");
  size_t smem = scatter_smem(PGX_OP_MIN_U32, nhubs);
  if (p.use_seg) smem = std::max(smem, seg_smem_bytes(p.seg.seg_log2) + 16);
  int grid = 0;
  void *args[] = {&p};
  void (*kern)(MinRunParams) =
      app == PGX_APP_SSSP
          ? (p.interleaved ? min_run_kernel<PGX_APP_SSSP, 1>
                           : bfs ? min_run_kernel<PGX_APP_SSSP, 0, true, false>
                                 : min_run_kernel<PGX_APP_SSSP, 0>)
          : (p.interleaved ? min_run_kernel<PGX_APP_CC, 1>
             : pre         ? min_run_kernel<PGX_APP_CC, 0, false, true, true>
                           : min_run_kernel<PGX_APP_CC, 0>);
  rc = coop_grid(kern, smem, &grid);
  if (rc) return rc;
  PGX_CUDA(cudaLaunchCooperativeKernel((void *)kern, grid, kBlock, args, smem, st));
  return PGX_OK;
}

int pgx_sssp_run(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
                 const void *graph_ws, const int32_t *hub_ids, int32_t nhubs, int32_t source,
                 int32_t max_supersteps, uint32_t *dist, void *run_ws, size_t run_ws_bytes,
                 int64_t *stats, uintptr_t stream) {
  return min_run(PGX_APP_SSSP, n, m, row_ptr, col_idx, graph_ws, hub_ids, nhubs, source,
                 max_supersteps, dist, run_ws, run_ws_bytes, stats, stream);
}

int pgx_sssp_run_ex(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
                    const void *graph_ws, const PgxSegIndex *seg, int32_t source,
                    int32_t max_supersteps, uint32_t *dist, void *run_ws, size_t run_ws_bytes,
                    int64_t *stats, uintptr_t stream) {
  return min_run(PGX_APP_SSSP, n, m, row_ptr, col_idx, graph_ws, nullptr, 0, source,
                 max_supersteps, dist, run_ws, run_ws_bytes, stats, stream, seg);
}

int pgx_sssp_run_dir(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
                     const void *graph_ws, const PgxSegIndex *seg, const int32_t *in_row_ptr,
                     const int32_t *in_col, int32_t source, int32_t max_supersteps,
                     uint32_t *dist, void *run_ws, size_t run_ws_bytes, int64_t *stats,
                     uintptr_t stream) {
  if (!in_row_ptr || (m > 0 && !in_col)) return fail(PGX_EINVAL, "null in-CSR pointer");
  if (reinterpret_cast<uintptr_t>(in_col) % 32)  // 256-bit sector loads (pgx_pull.cuh)
    return fail(PGX_EINVAL, "in_col must be 32-byte aligned");
  return min_run(PGX_APP_SSSP, n, m, row_ptr, col_idx, graph_ws, nullptr, 0, source,
                 max_supersteps, dist, run_ws, run_ws_bytes, stats, stream, seg, in_row_ptr,
                 in_col);
}

int pgx_cc_run_ex(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
                  const void *graph_ws, const PgxSegIndex *seg, int32_t max_supersteps,
                  uint32_t *labels, void *run_ws, size_t run_ws_bytes, int64_t *stats,
                  uintptr_t stream) {
  return min_run(PGX_APP_CC, n, m, row_ptr, col_idx, graph_ws, nullptr, 0, 0, max_supersteps,
                 labels, run_ws, run_ws_bytes, stats, stream, seg);
}

int pgx_cc_run_prescattered(int32_t n, int64_t m, const int32_t *row_ptr,
                            const int32_t *col_idx, const void *graph_ws,
                            int32_t max_supersteps, uint32_t *labels, void *run_ws,
                            size_t run_ws_bytes, int64_t *stats, uintptr_t stream) {
  return min_run(PGX_APP_CC, n, m, row_ptr, col_idx, graph_ws, nullptr, 0, 0, max_supersteps,
                 labels, run_ws, run_ws_bytes, stats, stream, nullptr, nullptr, nullptr, true);
}

int pgx_cc_run(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
               const void *graph_ws, const int32_t *hub_ids, int32_t nhubs,
               int32_t max_supersteps, uint32_t *labels, void *run_ws, size_t run_ws_bytes,
               int64_t *stats, uintptr_t stream) {
  return min_run(PGX_APP_CC, n, m, row_ptr, col_idx, graph_ws, hub_ids, nhubs, 0,
                 max_supersteps, labels, run_ws, run_ws_bytes, stats, stream);
}

#if PGX_COUNT_OPS
// debug build only: read and reset the scatter's operation counters
int pgx_debug_counts(unsigned long long *out) {
  PGX_CUDA(cudaDeviceSynchronize());
  PGX_CUDA(cudaMemcpyFromSymbol(out, g_pgx_ops, sizeof(unsigned long long) * 3));
  const unsigned long long z[3] = {0ull, 0ull, 0ull};
  PGX_CUDA(cudaMemcpyToSymbol(g_pgx_ops, z, sizeof z));
  return PGX_OK;
}
#endif

int pgx_hub_capacity(int32_t *capacity) {
  if (!capacity) return fail(PGX_EINVAL, "null out pointer");
  *capacity = kHubs;
  return PGX_OK;
}

int pgx_pagerank_run(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
                     const void *graph_ws, int32_t iterations, double damping, double base,
                     double r0, int32_t max_supersteps, double *rank, void *run_ws,
                     size_t run_ws_bytes, int64_t *stats, uintptr_t stream) {
  int rc = check_graph(n, m, row_ptr, col_idx, graph_ws);
  if (rc) return rc;
  if (iterations < 1) return fail(PGX_EINVAL, "iterations must be >= 1");
  if (!(damping >= 0.0 && damping <= 1.0)) return fail(PGX_EINVAL, "damping must be in [0, 1]");
  if (max_supersteps < 1) return fail(PGX_EINVAL, "superstep cap must be >= 1");
  if (!rank || !run_ws || !stats) return fail(PGX_EINVAL, "null output pointer");
  PrRunParams p;
  p.n = n;
  p.m = m;
  p.row_ptr = row_ptr;
  p.col = col_idx;
  graph_ws_layout(n, m, &p.g, (char *)graph_ws);
  if (run_ws_layout(PGX_APP_PAGERANK, n, m, max_supersteps, &p.ws, (char *)run_ws) > run_ws_bytes)
    return fail(PGX_ENOMEM, "run workspace too small");
  p.rank = rank;
  p.iterations = iterations;
  p.damping = damping;
  p.base = base;
  p.r0 = r0;
  p.max_steps = max_supersteps;
  p.stats = stats;
  cudaStream_t st = (cudaStream_t)stream;
  PGX_CUDA(cudaMemsetAsync(p.ws.bar, 0, 64, st));
  PGX_CUDA(cudaMemsetAsync(p.ws.misc, 0, 64, st));
  const size_t smem = scatter_smem_bytes(PGX_OP_SUM_F64);
  int grid = 0;
  rc = coop_grid(pagerank_run_kernel, smem, &grid);
  if (rc) return rc;
  void *args[] = {&p};
  PGX_CUDA(cudaLaunchCooperativeKernel((void *)pagerank_run_kernel, grid, kBlock, args, smem, st));
  return PGX_OK;
}

}  // extern "C"

namespace {
int pagerank_pull_launch(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *in_row_ptr,
                         const int32_t *in_col, const void *in_graph_ws,
                         const int32_t *hub_slot, int32_t nhubs, int32_t iterations,
                         double damping, double base, double r0, int32_t max_supersteps,
                         double *rank, void *run_ws, size_t run_ws_bytes, int64_t *stats,
                         uintptr_t stream) {
  int rc = check_graph(n, m, in_row_ptr, in_col, in_graph_ws);
  if (rc) return rc;
  if (!row_ptr) return fail(PGX_EINVAL, "null out-CSR offsets");
  if (reinterpret_cast<uintptr_t>(in_col) % 32)  // 256-bit id loads in the fold
    return fail(PGX_EINVAL, "in_col must be 32-byte aligned");
  if (nhubs < 0 || nhubs > kPrHubCap) return fail(PGX_EINVAL, "nhubs must be in [0, pgx_pr_hub_capacity()]");
  if (nhubs > 0 && !hub_slot) return fail(PGX_EINVAL, "null hub_slot");
  if (iterations < 1) return fail(PGX_EINVAL, "iterations must be >= 1");
  if (!(damping >= 0.0 && damping <= 1.0)) return fail(PGX_EINVAL, "damping must be in [0, 1]");
  if (max_supersteps < 1) return fail(PGX_EINVAL, "superstep cap must be >= 1");
  if (!rank || !run_ws || !stats) return fail(PGX_EINVAL, "null output pointer");
  PrPullParams p;
  p.n = n;
  p.m = m;
  p.row_ptr = row_ptr;
  p.in_row_ptr = in_row_ptr;
  p.in_col = in_col;
  graph_ws_layout(n, m, &p.gin, (char *)in_graph_ws);
  if (run_ws_layout(PGX_APP_PAGERANK_PULL, n, m, max_supersteps, &p.ws, (char *)run_ws) >
      run_ws_bytes)
    return fail(PGX_ENOMEM, "run workspace too small");
  p.rank = rank;
  p.iterations = iterations;
  p.damping = damping;
  p.base = base;
  p.r0 = r0;
  p.max_steps = max_supersteps;
  p.stats = stats;
  p.hub_slot = hub_slot;
  p.nhubs = nhubs;
  cudaStream_t st = (cudaStream_t)stream;
  PGX_CUDA(cudaMemsetAsync(p.ws.bar, 0, 64, st));
  PGX_CUDA(cudaMemsetAsync(p.ws.misc, 0, 64, st));
  const size_t smem = (size_t)kWarps * kSlots * 8 + 16 + (size_t)((nhubs + 1) & ~1) * 8;
  int grid = 0;
  void *args[] = {&p};
  if (nhubs > 0) {
    rc = coop_grid(pagerank_pull_kernel<true>, smem, &grid);
    if (rc) return rc;
    PGX_CUDA(cudaLaunchCooperativeKernel((void *)pagerank_pull_kernel<true>, grid, kBlock, args,
                                         smem, st));
  } else {
    rc = coop_grid(pagerank_pull_kernel<false>, smem, &grid);
    if (rc) return rc;
    PGX_CUDA(cudaLaunchCooperativeKernel((void *)pagerank_pull_kernel<false>, grid, kBlock, args,
                                         smem, st));
  }
  return PGX_OK;
}
}  // namespace

extern "C" {

int pgx_pr_hub_capacity(int32_t *capacity) {
  if (!capacity) return fail(PGX_EINVAL, "null output pointer");
  *capacity = kPrHubCap;
  return PGX_OK;
}

int pgx_pagerank_pull_run(int32_t n, int64_t m, const int32_t *row_ptr,
                          const int32_t *in_row_ptr, const int32_t *in_col,
                          const void *in_graph_ws, int32_t iterations, double damping,
                          double base, double r0, int32_t max_supersteps, double *rank,
                          void *run_ws, size_t run_ws_bytes, int64_t *stats, uintptr_t stream) {
  return pagerank_pull_launch(n, m, row_ptr, in_row_ptr, in_col, in_graph_ws, nullptr, 0,
                              iterations, damping, base, r0, max_supersteps, rank, run_ws,
                              run_ws_bytes, stats, stream);
}

int pgx_pagerank_pull_hubs_run(int32_t n, int64_t m, const int32_t *row_ptr,
                               const int32_t *in_row_ptr, const int32_t *in_col_hubs,
                               const void *in_graph_ws, const int32_t *hub_slot, int32_t nhubs,
                               int32_t iterations, double damping, double base, double r0,
                               int32_t max_supersteps, double *rank, void *run_ws,
                               size_t run_ws_bytes, int64_t *stats, uintptr_t stream) {
  return pagerank_pull_launch(n, m, row_ptr, in_row_ptr, in_col_hubs, in_graph_ws, hub_slot,
                              nhubs, iterations, damping, base, r0, max_supersteps, rank, run_ws,
                              run_ws_bytes, stats, stream);
}

}  // extern "C"
