// pgx_engine.cu -- B200 (sm_100a) push-superstep engine behind include/pgx.h.
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
//                       + one hardware atomicMin.u32 / red.add.f64; the
//                       unique lane that gets NEUTRAL back is the first
//                       publisher and appends the recipient to R (warp-
//                       aggregated), replacing the lock-protected publish.
//   externalisation  -> SoA: value[], mailbox[], frontier SoA, recipients.
//   edge-centric     -> the frontier is built with its exclusive edge
//                       prefix (one 64-bit packed atomic per warp); the
//                       scatter walks fixed 4096-edge tiles of that edge
//                       space, each CTA finds a tile's sources from a tile
//                       map and each edge's source by a shared-memory
//                       search -- exact edge balance, hub rows split.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <type_traits>

#include "../../include/pgx.h"

#ifndef PGX_MIN_BLOCKS
#define PGX_MIN_BLOCKS 2
#endif
#ifndef PGX_SCATTER_SMEM
#define PGX_SCATTER_SMEM 1   // stage each warp tile's sources in shared memory
#endif

namespace {

constexpr int kBlock = 512;          // threads per CTA
constexpr int kWarps = kBlock / 32;
constexpr int kItems = 8;            // 32-edge rounds per warp tile
constexpr int kTile = 32 * kItems;   // 256 edges per warp tile
#ifndef PGX_PASS
#define PGX_PASS 4
#endif
constexpr int kPass = PGX_PASS;      // rounds in flight per pass
constexpr int kSlots = kTile + 2;    // sources per warp tile (+ sentinel)
constexpr uint32_t kNeutralMin = 0xFFFFFFFFu;
constexpr int kHubs = 12288;         // hub recipients cached per CTA (48 KB smem)
constexpr int kInvalidEdge = 0x7FFFFFFF;  // never a vertex id (n < 2^31 - 1)
constexpr int kApplyListBytes = 128 * 32 * 4;  // apply: up to 128 words * 32 vertex ids
constexpr int kMaxCtas = 4096;
constexpr int kCompactBlock = 1024;

thread_local std::string g_last_error;

// tuning knobs (pgx_set_option); defaults are the shipped configuration
int g_opt[PGX_OPT_COUNT] = {
    /* PGX_OPT_READ_FILTER */ 1,
    /* PGX_OPT_CTAS_PER_SM */ 0,   // 0 = occupancy maximum
};

int fail(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char *what) {
  return fail(PGX_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define PGX_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);  \
  } while (0)

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ------------------------------------------------------------------
// device helpers
// ------------------------------------------------------------------

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// streamed, read-only neighbour ids: no L1 allocation, first to leave L2
__device__ __forceinline__ int ld_stream(const int *p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}


// 32-byte streamed load (sm_100: LDG.E.NA.ENL2.256) -- a warp reading
// 32 consecutive 32-byte chunks touches exactly 32 fully used sectors
__device__ __forceinline__ void ld_stream8(const int *p, uint64_t pol, int (&v)[8]) {
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, "
      "[%8], %9;"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "l"(p), "l"(pol));
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ void red_min_u32(uint32_t *p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.min.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void red_or_b32(uint32_t *p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ __attribute__((unused)) unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Sense-counting grid barrier for a co-resident (cooperative) grid.  The
// gpu-scope fences on both sides also invalidate L1 (CCTL.IVALL), so the
// weak, L1-cacheable mailbox reads of the next phase never see values
// from before the barrier.
struct GridBarrier {
  unsigned count;
  unsigned gen;
};

__device__ __forceinline__ void grid_sync(GridBarrier *bar, unsigned &gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned arrived = atomicAdd(&bar->count, 1u);
    if (arrived == gridDim.x - 1) {
      bar->count = 0;
      __threadfence();
      atomicExch(&bar->gen, gen + 1);
    } else {
      while (ld_acquire(&bar->gen) == gen) {
      }
    }
    __threadfence();
  }
  gen += 1;
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T *red) {
  // fixed-order tree: deterministic for a fixed block size
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
  if (lane_id() == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  T r = 0;
  if (threadIdx.x < 32) {
    r = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : T(0);
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xFFFFFFFFu, r, o);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

// ------------------------------------------------------------------
// workspace layouts
// ------------------------------------------------------------------

struct GraphWs {  // per graph, built once by pgx_graph_prepare
  int32_t *hdr;        // [0] = number of non-zero-degree vertices
  int32_t *nz_id;      // [n] ascending ids with out-degree > 0
  int32_t *nz_eb;      // [n+1] their row starts (= exclusive edge prefix)
  int32_t *tile_src;   // [ceil(m/kTile)+1] first nz index of each tile
  int32_t *blk;        // [ceil(n/kCompactBlock)+1] compaction scratch
};

size_t graph_ws_layout(int64_t n, int64_t m, GraphWs *ws, char *base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char *p = base ? base + off : nullptr;
    off += align_up(bytes);
    return p;
  };
  GraphWs w;
  w.hdr = (int32_t *)take(16);
  w.nz_id = (int32_t *)take(sizeof(int32_t) * (size_t)(n + 1));
  w.nz_eb = (int32_t *)take(sizeof(int32_t) * (size_t)(n + 1));
  w.tile_src = (int32_t *)take(sizeof(int32_t) * (size_t)(ceil_div(m, kTile) + 2));
  w.blk = (int32_t *)take(sizeof(int32_t) * (size_t)(ceil_div(n, kCompactBlock) + 2));
  if (ws) *ws = w;
  return off;
}

struct StepCounters {
  unsigned long long packed;  // senders << 32 | edges (frontier build)
  unsigned recip;             // recipients published by the scatter
  unsigned bcast;             // broadcasts (CC messages_sent)
  unsigned long long pad[2];
};

struct RunWs {
  GridBarrier *bar;        // zeroed by the host before every launch
  StepCounters *ctr;       // [max_supersteps + 2]
  double *partials;        // [kMaxCtas] PageRank dangling partial sums
  unsigned long long *misc;  // [0] dangling vertex count
  int32_t *f_eb;           // [n+1] frontier: exclusive edge prefix
  int32_t *f_rs;           // [n]   frontier: CSR row start
  void *f_msg;             // [n]   frontier: message (u32) / PR share (f64)
  uint32_t *has;           // [n/32+1] has-message bitmask (first publishers)
  int32_t *tile_src;       // [ceil(m/kTile)+2] sparse tile map
  void *mailbox;           // [n]   u32 (min) or f64 (sum); pull PR: folded sums
  double *share2;          // pull PR: second share buffer
  double *head, *tail;     // pull PR: per-tile partials of tile-spanning rows
};

size_t run_ws_layout(int app, int64_t n, int64_t m, int32_t max_steps, RunWs *ws,
                     char *base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char *p = base ? base + off : nullptr;
    off += align_up(bytes);
    return p;
  };
  const bool pr = app == PGX_APP_PAGERANK || app == PGX_APP_PAGERANK_PULL;
  const size_t W = pr ? 8 : 4;
  RunWs w;
  w.bar = (GridBarrier *)take(64);
  w.ctr = (StepCounters *)take(sizeof(StepCounters) * (size_t)(max_steps + 2));
  w.partials = (double *)take(sizeof(double) * kMaxCtas);
  w.misc = (unsigned long long *)take(64);
  w.f_msg = take(W * (size_t)(n + 1));
  w.mailbox = take(W * (size_t)(n + 1));
  w.share2 = w.head = w.tail = nullptr;
  if (app == PGX_APP_PAGERANK_PULL) {
    w.share2 = (double *)take(sizeof(double) * (size_t)(n + 1));
    w.head = (double *)take(sizeof(double) * (size_t)(ceil_div(m, kTile) + 2));
    w.tail = (double *)take(sizeof(double) * (size_t)(ceil_div(m, kTile) + 2));
  }
  if (!pr) {
    w.f_eb = (int32_t *)take(sizeof(int32_t) * (size_t)(n + 1));
    w.f_rs = (int32_t *)take(sizeof(int32_t) * (size_t)(n + 1));
    w.has = (uint32_t *)take(sizeof(uint32_t) * (size_t)(n / 32 + 2));
    w.tile_src = (int32_t *)take(sizeof(int32_t) * (size_t)(ceil_div(m, kTile) + 2));
  } else {
    w.f_eb = w.f_rs = w.tile_src = nullptr;
    w.has = nullptr;
  }
  if (ws) *ws = w;
  return off;
}

// ------------------------------------------------------------------
// the scatter phase: one pass of "every sender sends along its out-edges,
// messages combined into the recipient's mailbox slot"
// ------------------------------------------------------------------

enum class MsgSrc { kFrontier, kSourceId, kShareById };

struct ScatterArgs {
  const int32_t *col;     // col_idx
  const int32_t *eb;      // exclusive edge prefix per source
  const int32_t *rs;      // row start per source (sparse only)
  const int32_t *ids;     // vertex id per source (dense only)
  const void *msg;        // per-source message (sparse) / per-vertex share
  const int32_t *tile_src;  // source containing the first edge of each warp tile
  int32_t nsrc;           // number of sources
  int64_t E;              // edges in this pass
  void *mailbox;
  uint32_t *has;          // has-message bitmask (min only; nullptr: none)
  int32_t id_offset;      // kSourceId: message = ids[i] + id_offset
  const int32_t *hub_ids; // hub slot -> vertex; col_idx entries of hubs are
  int32_t nhubs;          // (sign bit | slot).  nhubs == 0: no hub cache
};

// shared memory of the scatter: one source window per warp (+ the hub
// cache of the min combiner, right after the windows)
__host__ __device__ constexpr size_t scatter_windows_smem(int op) {
  return PGX_SCATTER_SMEM
             ? (size_t)kWarps * kSlots * (sizeof(int32_t) * 2 + (op == PGX_OP_SUM_F64 ? 8 : 4))
             : (size_t)kApplyListBytes;  // the apply's recipient list still needs smem
}
__host__ __device__ constexpr size_t scatter_smem(int op, int nhubs = 0) {
  return scatter_windows_smem(op) + (op == PGX_OP_MIN_U32 ? sizeof(uint32_t) * nhubs : 0) + 16;
}

// One superstep's scatter.  Every warp owns whole 256-edge tiles of the
// senders' edge space (exact edge balance; a hub row spans many tiles) and
// runs without block barriers:
//   1. the tile map gives the source holding the tile's first edge; the
//      <= 257 sources of the tile are staged in the warp's smem window;
//   2. per round of 32 consecutive edges, lane j holds the start of
//      candidate source cur+1+j; the OR-reduction (REDUX) of the boundary
//      bits that fall in the window gives every lane its source with one
//      popc (sources have >= 1 edge, so <= 32 boundaries per window);
//   3. the 8 neighbour ids are streamed (L1::no_allocate, L2 evict_first),
//      then combined (min: read-filter + red.min, first publisher sets the
//      has-message bit; sum: red.add.f64).
// Hybrid combiner for hub recipients (the paper's split by recipient
// class): the top in-degree vertices are flagged in the encoded col_idx
// and filtered against a per-CTA shared-memory copy of their mailbox;
// only a CTA-local improvement goes to the global red.min.
#ifdef PGX_COUNT_OPS
__device__ unsigned long long g_dbg_reds, g_dbg_bits, g_dbg_edges;
#endif

template <int OP, MsgSrc MS>
__device__ void scatter_phase(const ScatterArgs &a, char *smem, bool read_filter = true) {
  using Msg = typename std::conditional<OP == PGX_OP_SUM_F64, double, uint32_t>::type;
  constexpr bool kDense = MS != MsgSrc::kFrontier;
  const int lane = (int)lane_id();
  const int warp = threadIdx.x >> 5;
  int32_t *s_eb = reinterpret_cast<int32_t *>(smem) + warp * kSlots;
  int32_t *s_rs = reinterpret_cast<int32_t *>(smem) + kWarps * kSlots + warp * kSlots;
  Msg *s_msg = reinterpret_cast<Msg *>(reinterpret_cast<int32_t *>(smem) + 2 * kWarps * kSlots) +
               warp * kSlots;
  const uint64_t pol = evict_first_policy();
  const int64_t ntiles = (a.E + kTile - 1) / kTile;
  const unsigned upto = (lane == 31) ? 0xFFFFFFFFu : ((2u << lane) - 1u);
  const int64_t gwarp = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  uint32_t *s_hub = reinterpret_cast<uint32_t *>(smem + scatter_windows_smem(OP));
  if (OP == PGX_OP_MIN_U32 && a.nhubs > 0) {  // block-uniform
    for (int i = threadIdx.x; i < a.nhubs; i += blockDim.x) s_hub[i] = kNeutralMin;
    __syncthreads();
  }

  for (int64_t t = gwarp; t < ntiles; t += nwarps) {
    const int64_t e0 = t * kTile;
    const int64_t e1 = min(a.E, e0 + kTile);
    const int i0 = a.tile_src[t];
    const int i1 = (t + 1 < ntiles) ? a.tile_src[t + 1] : a.nsrc - 1;
    const int k = i1 - i0 + 1;  // <= kTile + 1
#if PGX_SCATTER_SMEM
    __syncwarp();
    for (int j = lane; j <= k; j += 32) {
      const int i = i0 + j;
      if (j < k) {
        s_eb[j] = a.eb[i];
        if (!kDense) s_rs[j] = a.rs[i];
        if (MS == MsgSrc::kFrontier) {
          s_msg[j] = reinterpret_cast<const Msg *>(a.msg)[i];
        } else if (MS == MsgSrc::kSourceId) {
          s_msg[j] = (Msg)(a.ids[i] + a.id_offset);
        } else {
          s_msg[j] = reinterpret_cast<const Msg *>(a.msg)[a.ids[i]];
        }
      } else {
        s_eb[j] = (i < a.nsrc) ? a.eb[i] : (int32_t)a.E;  // sentinel
      }
    }
    __syncwarp();
#define PGX_EB(j) s_eb[j]
#define PGX_RS(j) s_rs[j]
#define PGX_MSG(j) s_msg[j]
#else
    // no staging: boundary candidates are 32 consecutive ints (one or two
    // sectors per round) and per-source data are broadcast loads, both
    // L1 hits after the first round -- all of shared memory stays L1
    const int32_t *g_eb = a.eb + i0;
    const int nrem = a.nsrc - i0;
#define PGX_EB(j) ((j) < nrem ? __ldg(g_eb + (j)) : (int32_t)a.E)
#define PGX_RS(j) __ldg(a.rs + i0 + (j))
#define PGX_MSG(j)                                                              \
  (MS == MsgSrc::kFrontier ? __ldg(reinterpret_cast<const Msg *>(a.msg) + i0 + (j)) \
   : MS == MsgSrc::kSourceId ? (Msg)(__ldg(a.ids + i0 + (j)) + a.id_offset)       \
   : __ldg(reinterpret_cast<const Msg *>(a.msg) + __ldg(a.ids + i0 + (j))))
#endif

    int cur = 0;  // eb[0] <= e0: tile_src names the source holding e0
#pragma unroll 1
    for (int pass = 0; pass < kItems / kPass; pass++) {
      int w[kPass];
      Msg mv[kPass];
#pragma unroll
      for (int r = 0; r < kPass; r++) {
        const int64_t base = e0 + (pass * kPass + r) * 32;
        const int64_t e = base + lane;
        const int ci = cur + 1 + lane;
        unsigned bit = 0;
        if (ci <= k) {
          const int64_t pp = (int64_t)PGX_EB(ci) - base;
          if (pp >= 0 && pp < 32) bit = 1u << pp;
        }
        const unsigned bm = __reduce_or_sync(0xFFFFFFFFu, bit);
        const int src = cur + __popc(bm & upto);
        cur += __popc(bm);
        w[r] = kInvalidEdge;
        if (e < e1) {
          const int64_t pos = kDense ? e : (int64_t)PGX_RS(src) + (e - PGX_EB(src));
          w[r] = ld_stream(a.col + pos, pol);
          mv[r] = PGX_MSG(src);
        }
      }
      if (OP == PGX_OP_MIN_U32) {
        // hybrid combiner, fire-and-forget: read-filter (the mailbox.py:159
        // short-circuit), then one red.min.u32.  Publication (mailbox.py:
        // 190-199) becomes an idempotent has-message bit set by every lane
        // whose filter read saw NEUTRAL: the lane whose atomic lands first
        // on an empty slot necessarily read NEUTRAL, so no recipient is
        // lost, and nothing waits on an atomic's return value.
        uint32_t *mb = reinterpret_cast<uint32_t *>(a.mailbox);
        uint32_t old[kPass];
#pragma unroll
        for (int r = 0; r < kPass; r++) {
          const int x = w[r];
          old[r] = (x == kInvalidEdge) ? 0u
                   : (x < 0) ? s_hub[x & 0x7FFFFFFF]  // hub: CTA-local filter
                   : (read_filter ? mb[x] : kNeutralMin);
        }
#pragma unroll
        for (int r = 0; r < kPass; r++) {
          const int x = w[r];
          const uint32_t msg = (uint32_t)mv[r];
          if (x != kInvalidEdge && msg < old[r]) {
            int v = x;
            uint32_t prev = old[r];
            if (x < 0) {  // hub: the CTA-local copy let it through; consult
                          // the global slot (the shared filter) before the red
              const int slot = x & 0x7FFFFFFF;
              v = a.hub_ids[slot];
              prev = mb[v];
              s_hub[slot] = min(prev, msg);  // racy store: only weakens the filter
              if (msg >= prev) v = -1;
            }
            if (v >= 0) {
              red_min_u32(mb + v, msg);
              if (a.has && prev == kNeutralMin) red_or_b32(a.has + (v >> 5), 1u << (v & 31));
#ifdef PGX_COUNT_OPS
              atomicAdd(&g_dbg_reds, 1ull);
              if (prev == kNeutralMin) atomicAdd(&g_dbg_bits, 1ull);
#endif
            }
          }
#ifdef PGX_COUNT_OPS
          if (x != kInvalidEdge) atomicAdd(&g_dbg_edges, 1ull);
#endif
        }
      } else {
        double *mb = reinterpret_cast<double *>(a.mailbox);
#pragma unroll
        for (int r = 0; r < kPass; r++)
          if (w[r] != kInvalidEdge) atomicAdd(mb + w[r], (double)mv[r]);
      }
    }
#undef PGX_EB
#undef PGX_RS
#undef PGX_MSG
  }
}

// ------------------------------------------------------------------
// sparse apply for the min programs (SSSP / CC), driven by the
// has-message bitmask: consume every flagged mailbox (vertex order),
// adopt an improvement, append improved vertices to the next frontier
// with their edge prefix.  One 64-bit atomic per block chunk reserves
// (frontier slots, edge range); the tile map is written as a side effect.
// ------------------------------------------------------------------

__device__ __forceinline__ unsigned long long block_excl_scan_u64(unsigned long long x,
                                                                  unsigned long long *s_w,
                                                                  unsigned long long *total) {
  unsigned long long incl = x;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if ((int)lane_id() >= o) incl += y;
  }
  if (lane_id() == 31) s_w[threadIdx.x >> 5] = incl;
  __syncthreads();
  if (threadIdx.x < 32) {
    const unsigned long long w = (threadIdx.x < kWarps) ? s_w[threadIdx.x] : 0ull;
    unsigned long long wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if ((int)threadIdx.x >= o) wi += y;
    }
    if (threadIdx.x < kWarps) s_w[threadIdx.x] = wi - w;
    if (threadIdx.x == 31) s_w[32] = wi;
  }
  __syncthreads();
  const unsigned long long r = s_w[threadIdx.x >> 5] + incl - x;
  *total = s_w[32];
  __syncthreads();
  return r;
}

// Apply chunk: kApplyWords bitmask words per block iteration.  The set
// bits are first compacted into a shared-memory vertex list (block scan
// of popcounts), then every thread consumes up to kApplyItems recipients
// with independent loads -- no per-word serial chains.
#ifndef PGX_APPLY_WORDS
#define PGX_APPLY_WORDS 64
#endif
constexpr int kApplyWords = PGX_APPLY_WORDS;
constexpr int kApplyItems = kApplyWords * 32 / kBlock;  // 4

// Returns (recipients counted) << 32 | (broadcasts) for this thread.  With
// `count_only` the bitmask is only counted (superstep cap reached: the
// pending messages must stay unconsumed, engine.py:299-300).
template <int APP>
__device__ unsigned long long apply_min_phase(const int32_t *__restrict__ row_ptr, uint32_t *val,
                                              uint32_t *mailbox, int32_t n, const RunWs &ws,
                                              StepCounters *ctr, char *smem, bool count_only) {
  __shared__ unsigned long long s_w[33];
  __shared__ unsigned long long s_gbase;
  int32_t *s_list = reinterpret_cast<int32_t *>(smem);  // kApplyWords * 32 ids
  uint32_t *f_msg = reinterpret_cast<uint32_t *>(ws.f_msg);
  const int words = (n + 31) >> 5;
  unsigned bcast = 0, recips = 0;
  if (count_only) {
    for (int wi = blockIdx.x * kBlock + threadIdx.x; wi < words; wi += gridDim.x * kBlock)
      recips += __popc(ws.has[wi]);
    return ((unsigned long long)recips << 32);
  }
  for (int base = blockIdx.x * kApplyWords; base < words; base += gridDim.x * kApplyWords) {
    // ---- expand the chunk's set bits into s_list (vertex order) ----
    uint32_t word = 0;
    const int wi = base + threadIdx.x;
    if (threadIdx.x < kApplyWords && wi < words) {
      word = ws.has[wi];
      if (word) ws.has[wi] = 0u;
    }
    if (!__syncthreads_or(word != 0)) continue;  // empty chunk: one barrier
    recips += __popc(word);
    unsigned long long tot64;
    const int off = (int)block_excl_scan_u64((unsigned long long)__popc(word), s_w, &tot64);
    const int T = (int)tot64;
    if (T == 0) continue;  // block-uniform
    {
      int o = off;
      uint32_t rem = word;
      while (rem) {
        const int b = __ffs(rem) - 1;
        rem &= rem - 1;
        s_list[o++] = (wi << 5) + b;
      }
    }
    __syncthreads();
    // ---- consume + compute, kApplyItems independent recipients / thread ----
    int v[kApplyItems];
    uint32_t m[kApplyItems], cv[kApplyItems];
    int deg[kApplyItems], rs[kApplyItems];
#pragma unroll
    for (int j = 0; j < kApplyItems; j++) {
      const int idx = j * kBlock + threadIdx.x;
      v[j] = (idx < T) ? s_list[idx] : -1;
    }
#pragma unroll
    for (int j = 0; j < kApplyItems; j++) {
      if (v[j] >= 0) {
        m[j] = mailbox[v[j]];
        cv[j] = val[v[j]];
      }
    }
    unsigned long long mine = 0;
#pragma unroll
    for (int j = 0; j < kApplyItems; j++) {
      deg[j] = 0;
      if (v[j] >= 0) {
        mailbox[v[j]] = kNeutralMin;  // consume (mailbox.py:112-117)
        if (m[j] < cv[j]) {
          val[v[j]] = m[j];
          bcast++;
          rs[j] = row_ptr[v[j]];
          deg[j] = -1;  // improved; degree resolved below
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kApplyItems; j++) {
      if (deg[j] == -1) {
        deg[j] = row_ptr[v[j] + 1] - rs[j];
        if (deg[j] > 0) mine += (1ull << 32) | (unsigned long long)deg[j];
      }
    }
    unsigned long long total;
    unsigned long long run = block_excl_scan_u64(mine, s_w, &total);
    if (total != 0) {  // block-uniform
      if (threadIdx.x == 0) s_gbase = atomicAdd(&ctr->packed, total);
      __syncthreads();
      run += s_gbase;
#pragma unroll
      for (int j = 0; j < kApplyItems; j++) {
        if (deg[j] > 0) {
          const unsigned pos = (unsigned)(run >> 32);
          const int eb = (int)(run & 0xFFFFFFFFull);
          ws.f_eb[pos] = eb;
          ws.f_rs[pos] = rs[j];
          f_msg[pos] = (APP == PGX_APP_SSSP) ? m[j] + 1u : m[j];
          for (int64_t t = ((int64_t)eb + kTile - 1) / kTile; t * kTile < (int64_t)eb + deg[j]; t++)
            ws.tile_src[t] = (int)pos;
          run += (1ull << 32) | (unsigned long long)deg[j];
        }
      }
    }
    __syncthreads();  // s_list / s_gbase reuse
  }
  return ((unsigned long long)recips << 32) | bcast;
}

__device__ __forceinline__ void record_step(int64_t *stats, int s, int64_t active,
                                            int64_t sent, int64_t edges, int64_t senders,
                                            int64_t recips, int64_t bcast) {
  int64_t *st = stats + PGX_STAT_HDR + (int64_t)s * PGX_STAT_FIELDS;
  st[0] = active;
  st[1] = sent;
  st[2] = edges;
  st[3] = senders;
  st[4] = recips;
  st[5] = (int64_t)globaltimer();
  st[6] = bcast;
}

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
  const int32_t *hub_ids;
  int32_t nhubs;
  int64_t *stats;
};

template <int APP>
__global__ void __launch_bounds__(kBlock, PGX_MIN_BLOCKS) min_run_kernel(MinRunParams p) {
  extern __shared__ __align__(16) char smem[];
  __shared__ unsigned s_red[32];
  unsigned gen = 0;
  if (threadIdx.x == 0) gen = ld_acquire(&p.ws.bar->gen);
  uint32_t *mailbox = reinterpret_cast<uint32_t *>(p.ws.mailbox);
  const unsigned nthreads = gridDim.x * blockDim.x;
  const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;

  // ---- setup (algorithms.py:96-97 / 129-134) + superstep-0 senders ----
  for (unsigned v = gtid; v < (unsigned)p.n; v += nthreads) {
    p.val[v] = (APP == PGX_APP_CC) ? v : kNeutralMin;
    mailbox[v] = kNeutralMin;
  }
  for (unsigned wi = gtid; wi < (unsigned)(p.n / 32 + 2); wi += nthreads) p.ws.has[wi] = 0u;
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
  grid_sync(p.ws.bar, gen);
  if (APP == PGX_APP_SSSP && gtid == 0) p.val[p.source] = 0u;
  if (gtid == 0) p.stats[PGX_STAT_HDR + 7] = (int64_t)globaltimer();

  for (int s = 0;; s++) {
    // ---- scatter(s): senders push along out-edges into the mailbox ----
    ScatterArgs a;
    a.col = p.col;
    a.mailbox = mailbox;
    a.has = p.ws.has;
    a.id_offset = 0;
    a.hub_ids = p.hub_ids;
    a.nhubs = p.nhubs;
    if (APP == PGX_APP_CC && s == 0) {
      a.eb = p.g.nz_eb;
      a.rs = nullptr;
      a.ids = p.g.nz_id;
      a.msg = nullptr;
      a.tile_src = p.g.tile_src;
      a.nsrc = p.g.hdr[0];
      a.E = p.m;
      scatter_phase<PGX_OP_MIN_U32, MsgSrc::kSourceId>(a, smem, p.read_filter);
    } else {
      const unsigned long long packed = p.ws.ctr[s].packed;
      a.eb = p.ws.f_eb;
      a.rs = p.ws.f_rs;
      a.ids = nullptr;
      a.msg = p.ws.f_msg;
      a.tile_src = p.ws.tile_src;
      a.nsrc = (int32_t)(packed >> 32);
      a.E = (int64_t)(packed & 0xFFFFFFFFull);
      scatter_phase<PGX_OP_MIN_U32, MsgSrc::kFrontier>(a, smem, p.read_filter);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      StepCounters z = {};
      p.ws.ctr[s + 1] = z;
    }
    grid_sync(p.ws.bar, gen);
    const uint64_t t_scatter = globaltimer();

    // ---- apply(s+1): consume + compute + frontier build; at the cap the
    //      pending messages are only counted (engine.py:299-300) ----
    const bool at_cap = (s + 1 == p.max_steps);
    const unsigned long long rb =
        apply_min_phase<APP>(p.row_ptr, p.val, mailbox, p.n, p.ws, &p.ws.ctr[s + 1], smem, at_cap);
    const unsigned bc = block_sum<unsigned>((unsigned)(rb & 0xFFFFFFFFull), s_red);
    const unsigned rc = block_sum<unsigned>((unsigned)(rb >> 32), s_red);
    if (threadIdx.x == 0) {
      if (bc) atomicAdd(&p.ws.ctr[s + 1].bcast, bc);
      if (rc) atomicAdd(&p.ws.ctr[s].recip, rc);
    }
    grid_sync(p.ws.bar, gen);

    // ---- stats + halt test (engine.py:284-300) ----
    const unsigned nrecip = p.ws.ctr[s].recip;
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

// ------------------------------------------------------------------
// pull-mode PageRank: the reference's own communication mode for PR
// (algorithms.py:80, engine.py:425-457).  A vertex folds the shares of its
// in-neighbours; no atomics at all.  The in-CSR edge space is walked in
// the same 256-edge warp tiles as the scatter (exact edge balance), with
// a segmented warp scan per 32-edge round.  Rows that fit in one tile are
// summed in-register and stored; rows spanning tiles leave per-tile
// partials (tail of the first tile, head of every later tile) that the
// apply combines in tile order -- deterministic for a fixed tiling.
// ------------------------------------------------------------------

struct GatherArgs {
  const int32_t *in_col;
  const int32_t *eb;        // in-row starts of vertices with in-degree > 0
  const int32_t *ids;       // those vertices
  const int32_t *tile_src;  // in-edge tile map
  int32_t nsrc;
  int64_t E;
  const double *share;      // shares broadcast last superstep
  double *folded, *head, *tail;
};

__device__ void gather_phase(const GatherArgs &a, char *smem) {
  const int lane = (int)lane_id();
  const int warp = threadIdx.x >> 5;
  int32_t *s_eb = reinterpret_cast<int32_t *>(smem) + warp * kSlots;
  int32_t *s_id = reinterpret_cast<int32_t *>(smem) + kWarps * kSlots + warp * kSlots;
  const uint64_t pol = evict_first_policy();
  const int64_t ntiles = (a.E + kTile - 1) / kTile;
  const int64_t gwarp = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t nwarps = (int64_t)gridDim.x * kWarps;

  for (int64_t t = gwarp; t < ntiles; t += nwarps) {
    const int64_t e0 = t * kTile;
    const int64_t e1 = min(a.E, e0 + kTile);
    const int i0 = a.tile_src[t];
    const int i1 = (t + 1 < ntiles) ? a.tile_src[t + 1] : a.nsrc - 1;
    const int k = i1 - i0 + 1;
    __syncwarp();
    for (int j = lane; j <= k; j += 32) {
      const int i = i0 + j;
      if (j < k) {
        s_eb[j] = a.eb[i];
        s_id[j] = a.ids[i];
      } else {
        s_eb[j] = (i < a.nsrc) ? a.eb[i] : (int32_t)a.E;
      }
    }
    __syncwarp();
    const bool first_open = (int64_t)s_eb[0] < e0;  // row began in an earlier tile
    // Each lane owns 8 contiguous in-edges [a0, a1): two 16-byte id loads,
    // 8 independent share gathers, a sequential per-row sum; one segmented
    // warp scan per tile carries partial rows across lanes.
    const int64_t a0 = e0 + 8 * lane;
    const int64_t a1 = min(e1, a0 + 8);
    const bool active = a0 < e1;
    int col[8];
    if (active && a1 - a0 == 8) {
      ld_stream8(a.in_col + a0, pol, col);
    } else {
#pragma unroll
      for (int j = 0; j < 8; j++) col[j] = (a0 + j < a1) ? ld_stream(a.in_col + a0 + j, pol) : -1;
    }
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; j++) x[j] = (col[j] >= 0) ? __ldg(a.share + col[j]) : 0.0;
    // row holding a0: largest idx with s_eb[idx] <= a0 (binary search over
    // the <= 258 staged row starts), then the starts of the next 8 rows as
    // a boundary bitmask over the lane's 9 positions a0..a0+8, so the walk
    // below runs on registers only
    int cur = 0;
    unsigned bmask = 0;
    if (active) {
      int hi = k;
      while (hi - cur > 1) {
        const int mid = (cur + hi) >> 1;
        if ((int64_t)s_eb[mid] <= a0) cur = mid; else hi = mid;
      }
#pragma unroll
      for (int i = 1; i <= 8; i++) {
        if (cur + i <= k) {
          const int64_t p = (int64_t)s_eb[cur + i] - a0;  // > 0 by construction
          if (p <= 8) bmask |= 1u << p;
        }
      }
    }
    const int first_seg = cur;
    bool first_closed = false;
    double first_part = 0.0, acc = 0.0;
#pragma unroll
    for (int j = 0; j <= 8; j++) {
      const int64_t e = a0 + j;
      if (!active || e > a1) break;
      if ((bmask >> j) & 1u) {  // the next row starts at e (e == a1: range end)
        if (cur == first_seg) {
          first_closed = true;
          first_part = acc;
        } else {
          a.folded[s_id[cur]] = acc;  // row lies inside this lane's range
        }
        cur++;
        acc = 0.0;
      }
      if (e < a1) acc = __dadd_rn(acc, x[j]);
    }
    // segmented inclusive scan of the open-row partials, keyed by row
    const int key = active ? cur : (1 << 30);
    double v = active ? acc : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xFFFFFFFFu, v, o);
      const int ko = __shfl_up_sync(0xFFFFFFFFu, key, o);
      if (lane >= o && ko == key) v = __dadd_rn(y, v);
    }
    const double prev_v = __shfl_up_sync(0xFFFFFFFFu, v, 1);
    const int prev_key = __shfl_up_sync(0xFFFFFFFFu, key, 1);
    const double carry_in = (lane > 0 && prev_key == first_seg) ? prev_v : 0.0;
    if (active) {
      if (first_closed) {  // this lane ends a row that began to its left
        const double tot = __dadd_rn(carry_in, first_part);
        if (first_seg == 0 && first_open) a.head[t] = tot;
        else a.folded[s_id[first_seg]] = tot;
      }
      if (a1 == e1 && cur < k && (int64_t)s_eb[cur] < e1) {
        // the tile ends inside row `cur`, which continues into the next tile
        const double tot = (cur == first_seg) ? __dadd_rn(carry_in, acc) : acc;
        if (cur == 0 && first_open) a.head[t] = tot;
        else a.tail[t] = tot;
      }
    }
  }
}

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
};

__global__ void __launch_bounds__(kBlock, PGX_MIN_BLOCKS) pagerank_pull_kernel(PrPullParams p) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double s_red[32];
  __shared__ unsigned long long s_ured[32];
  __shared__ double s_dangling;
  unsigned gen = 0;
  double *folded = reinterpret_cast<double *>(p.ws.mailbox);
  double *share_cur = reinterpret_cast<double *>(p.ws.f_msg);
  double *share_nxt = p.ws.share2;
  const unsigned nthreads = gridDim.x * blockDim.x;
  const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int last = p.iterations - 1;
  const double dn_n = (double)p.n;

  // ---- setup (algorithms.py:44-59): rank = r0, seed shares r0/outdeg ----
  unsigned long long my_dangling = 0;
  for (unsigned v = gtid; v < (unsigned)p.n; v += nthreads) {
    const int deg = p.row_ptr[v + 1] - p.row_ptr[v];
    p.rank[v] = p.r0;
    share_cur[v] = deg ? __ddiv_rn(p.r0, (double)deg) : 0.0;
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

  for (int s = 0;; s++) {
    if (blockIdx.x == 0 && threadIdx.x == 0)
      p.stats[PGX_STAT_HDR + (int64_t)s * PGX_STAT_FIELDS + 7] = (int64_t)globaltimer();
    // ---- fold (engine.py:425-457): in-neighbour shares of last superstep
    g.share = share_cur;
    gather_phase(g, smem);
    grid_sync(p.ws.bar, gen);
    const uint64_t t_fold = globaltimer();

    // ---- compute (algorithms.py:61-73): rank, next share, dangling mass
    const double dn = __ddiv_rn(dangling, dn_n);
    double my_d = 0.0;
    for (unsigned v = gtid; v < (unsigned)p.n; v += nthreads) {
      const int es = p.in_row_ptr[v], ee = p.in_row_ptr[v + 1];
      double f = 0.0;
      if (ee > es) {
        const int64_t t0 = es / kTile, t1 = (ee - 1) / kTile;
        if (t0 == t1) {
          f = folded[v];
        } else {
          f = p.ws.tail[t0];
          for (int64_t t = t0 + 1; t <= t1; t++) f = __dadd_rn(f, p.ws.head[t]);
        }
      }
      const double r = __dadd_rn(p.base, __dmul_rn(p.damping, __dadd_rn(f, dn)));
      p.rank[v] = r;
      const int deg = p.row_ptr[v + 1] - p.row_ptr[v];
      if (deg == 0) my_d = __dadd_rn(my_d, r);
      else if (s != last) share_nxt[v] = __ddiv_rn(r, (double)deg);
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
  }
}

// ------------------------------------------------------------------
// phase kernels of the partitioned (multi-GPU) superstep, SURVEY 8(e).
// Each rank owns the out-edges of a contiguous vertex range [lo, lo+len)
// and a slice of the mailbox.  Per superstep: K1 scatters the rank's
// senders into a FULL-WIDTH local mailbox (global destination ids); the
// host reduces the mailbox slices onto their owners (NCCL min / sum);
// K2 applies on the owned slice (has-message == mailbox != neutral after
// the min reduction: messages are < n <= 2^31 and never the neutral).
// Regular (non-cooperative) stream-ordered launches.
// ------------------------------------------------------------------

struct SliceCounters {       // device counters of one partitioned superstep
  unsigned long long packed; // senders << 32 | edges of the next frontier
  unsigned long long recip;  // recipients in the owned slice
  unsigned long long bcast;  // vertices that computed a new value
  double dangling;           // PageRank: rank mass of owned dangling vertices
};

#ifndef PGX_SCATTER_MIN_BLOCKS
#define PGX_SCATTER_MIN_BLOCKS PGX_MIN_BLOCKS
#endif

template <int OP, MsgSrc MS>
__global__ void __launch_bounds__(kBlock, PGX_SCATTER_MIN_BLOCKS) scatter_kernel(ScatterArgs a,
                                                                          int read_filter) {
  extern __shared__ __align__(16) char smem[];
  scatter_phase<OP, MS>(a, smem, read_filter != 0);
}

template <int APP>
__global__ void __launch_bounds__(kBlock) apply_slice_kernel(
    int32_t len, const int32_t *__restrict__ row_ptr, uint32_t *val, uint32_t *mailbox,
    int32_t *f_eb, int32_t *f_rs, uint32_t *f_msg, int32_t *tile_src, SliceCounters *ctr,
    int32_t count_only, uint32_t neutral) {
  __shared__ unsigned long long s_w[33];
  __shared__ unsigned long long s_gbase;
  __shared__ unsigned long long s_red[32];
  constexpr int kI = 4;
  const int base = blockIdx.x * kBlock * kI;
  int deg[kI], rs[kI];
  uint32_t m[kI];
  unsigned long long mine = 0, recips = 0, bcast = 0;
#pragma unroll
  for (int j = 0; j < kI; j++) {
    const int v = base + j * kBlock + threadIdx.x;
    deg[j] = 0;
    m[j] = (v < len) ? mailbox[v] : neutral;
    if (m[j] != neutral) {
      recips++;
      if (!count_only) {
        mailbox[v] = neutral;  // consume
        if (m[j] < val[v]) {
          val[v] = m[j];
          bcast++;
          rs[j] = row_ptr[v];
          deg[j] = row_ptr[v + 1] - rs[j];
          if (deg[j] > 0) mine += (1ull << 32) | (unsigned long long)deg[j];
        }
      }
    }
  }
  unsigned long long total;
  unsigned long long run = block_excl_scan_u64(mine, s_w, &total);
  if (total) {
    if (threadIdx.x == 0) s_gbase = atomicAdd(&ctr->packed, total);
    __syncthreads();
    run += s_gbase;
#pragma unroll
    for (int j = 0; j < kI; j++) {
      if (deg[j] > 0) {
        const unsigned pos = (unsigned)(run >> 32);
        const int eb = (int)(run & 0xFFFFFFFFull);
        f_eb[pos] = eb;
        f_rs[pos] = rs[j];
        f_msg[pos] = (APP == PGX_APP_SSSP) ? m[j] + 1u : m[j];
        for (int64_t t = ((int64_t)eb + kTile - 1) / kTile; t * kTile < (int64_t)eb + deg[j]; t++)
          tile_src[t] = (int)pos;
        run += (1ull << 32) | (unsigned long long)deg[j];
      }
    }
  }
  recips = block_sum<unsigned long long>(recips, s_red);
  if (threadIdx.x == 0 && recips) atomicAdd(&ctr->recip, recips);
  bcast = block_sum<unsigned long long>(bcast, s_red);
  if (threadIdx.x == 0 && bcast) atomicAdd(&ctr->bcast, bcast);
}

__global__ void __launch_bounds__(kBlock) pr_apply_slice_kernel(
    int32_t len, const int32_t *__restrict__ row_ptr, double *rank, double *mailbox,
    double *share, double base, double damping, double dn, int32_t last, double *partials) {
  __shared__ double s_red[32];
  const int v = blockIdx.x * kBlock + threadIdx.x;
  double my_d = 0.0;
  if (v < len) {
    const double folded = mailbox[v];
    mailbox[v] = 0.0;
    const double r = __dadd_rn(base, __dmul_rn(damping, __dadd_rn(folded, dn)));
    rank[v] = r;
    const int deg = row_ptr[v + 1] - row_ptr[v];
    if (deg == 0) my_d = r;
    else if (!last) share[v] = __ddiv_rn(r, (double)deg);
  }
  const double b = block_sum<double>(my_d, s_red);
  if (threadIdx.x == 0) partials[blockIdx.x] = b;
}

__global__ void slice_init_kernel(int app, int32_t len, int32_t lo, uint32_t *val,
                                  const int32_t *row_ptr, double *rank, double *share,
                                  double r0) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < len; v += gridDim.x * blockDim.x) {
    if (app == PGX_APP_CC) val[v] = (uint32_t)(lo + v);
    else if (app == PGX_APP_SSSP) val[v] = kNeutralMin;
    else {
      const int deg = row_ptr[v + 1] - row_ptr[v];
      rank[v] = r0;
      share[v] = deg ? __ddiv_rn(r0, (double)deg) : 0.0;
    }
  }
}

// ------------------------------------------------------------------
// graph preparation kernels: order-preserving compaction of the vertices
// with out-degree > 0 (warp ballot + block scan), then the tile map
// ------------------------------------------------------------------

__global__ void offsets_to_i32_kernel(const int64_t *in, int32_t *out, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)in[i];
}

__device__ __forceinline__ int block_excl_scan(int x, int *s_warp, int *total) {
  int incl = x;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if ((int)lane_id() >= o) incl += y;
  }
  if (lane_id() == 31) s_warp[threadIdx.x >> 5] = incl;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    int w = (threadIdx.x < nw) ? s_warp[threadIdx.x] : 0;
    int wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if ((int)threadIdx.x >= o) wi += y;
    }
    if (threadIdx.x < nw) s_warp[threadIdx.x] = wi - w;
    if (threadIdx.x == 31) s_warp[32] = wi;
  }
  __syncthreads();
  const int r = s_warp[threadIdx.x >> 5] + incl - x;
  *total = s_warp[32];
  __syncthreads();
  return r;
}

__global__ void nz_count_kernel(const int32_t *row_ptr, int32_t n, int32_t *blk) {
  __shared__ int s_warp[33];
  const int64_t v = blockIdx.x * (int64_t)kCompactBlock + threadIdx.x;
  const int f = (v < n && row_ptr[v + 1] > row_ptr[v]) ? 1 : 0;
  int total;
  block_excl_scan(f, s_warp, &total);
  if (threadIdx.x == 0) blk[blockIdx.x] = total;
}

__global__ void nz_scan_blocks_kernel(int32_t *blk, int32_t nb, int32_t *hdr) {
  // single CTA: exclusive scan of per-block counts
  __shared__ int s_warp[33];
  int carry = 0;
  for (int base = 0; base < nb; base += kCompactBlock) {
    const int i = base + threadIdx.x;
    const int x = (i < nb) ? blk[i] : 0;
    int total;
    const int ex = block_excl_scan(x, s_warp, &total);
    if (i < nb) blk[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) {
    blk[nb] = carry;
    hdr[0] = carry;
  }
}

__global__ void nz_write_kernel(const int32_t *row_ptr, int32_t n, const int32_t *blk,
                                int32_t *nz_id, int32_t *nz_eb, int64_t m) {
  __shared__ int s_warp[33];
  const int64_t v = blockIdx.x * (int64_t)kCompactBlock + threadIdx.x;
  const int f = (v < n && row_ptr[v + 1] > row_ptr[v]) ? 1 : 0;
  int total;
  const int ex = block_excl_scan(f, s_warp, &total);
  if (f) {
    const int pos = blk[blockIdx.x] + ex;
    nz_id[pos] = (int32_t)v;
    nz_eb[pos] = row_ptr[v];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) nz_eb[blk[gridDim.x]] = (int32_t)m;
}

__global__ void tile_map_kernel(const int32_t *hdr, const int32_t *nz_eb, int32_t *tile_src) {
  const int nnz = hdr[0];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += gridDim.x * blockDim.x) {
    const int64_t eb = nz_eb[i], ee = nz_eb[i + 1];
    for (int64_t t = (eb + kTile - 1) / kTile; t * kTile < ee; t++) tile_src[t] = i;
  }
}

// ------------------------------------------------------------------
// R-MAT generator, input construction only
// ------------------------------------------------------------------

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void rmat_kernel(int scale, int64_t first, int64_t count, uint64_t ta, uint64_t tab,
                            uint64_t tabc, uint64_t base, int symmetric, int64_t lo, int64_t hi,
                            unsigned long long *keys, int64_t capacity,
                            unsigned long long *counter) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t i = (uint64_t)(first + k);
    uint64_t s = 0, d = 0;
    for (int l = 0; l < scale; l++) {
      const uint64_t r = splitmix64(base + i * (uint64_t)scale + (uint64_t)l) >> 11;
      const int q = r < ta ? 0 : r < tab ? 1 : r < tabc ? 2 : 3;
      const int bit = scale - 1 - l;
      s |= (uint64_t)(q >> 1) << bit;
      d |= (uint64_t)(q & 1) << bit;
    }
    if (s == d) continue;
    const bool fwd = (int64_t)s >= lo && (int64_t)s < hi;
    const bool rev = symmetric && (int64_t)d >= lo && (int64_t)d < hi;
    const int cnt = (fwd ? 1 : 0) + (rev ? 1 : 0);
    if (!cnt) continue;
    unsigned long long pos = atomicAdd(counter, (unsigned long long)cnt);
    if (fwd && (int64_t)pos < capacity) keys[pos++] = (s << 32) | d;
    if (rev && (int64_t)pos < capacity) keys[pos] = (d << 32) | s;
  }
}

// ------------------------------------------------------------------
// launch helpers
// ------------------------------------------------------------------

size_t scatter_smem_bytes(int op) { return scatter_smem(op); }

template <typename K>
int coop_grid(K kernel, size_t smem, int *grid) {
  int dev = 0, sms = 0, per_sm = 0;
  PGX_CUDA(cudaGetDevice(&dev));
  PGX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  PGX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  PGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, smem));
  if (per_sm < 1) return fail(PGX_ECUDA, "persistent kernel does not fit on an SM");
  if (g_opt[PGX_OPT_CTAS_PER_SM] > 0 && g_opt[PGX_OPT_CTAS_PER_SM] < per_sm)
    per_sm = g_opt[PGX_OPT_CTAS_PER_SM];
  int g = sms * per_sm;
  if (g > kMaxCtas) g = kMaxCtas;
  *grid = g;
  return PGX_OK;
}

int check_graph(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
                const void *graph_ws) {
  if (n < 1) return fail(PGX_EINVAL, "vertex count must be >= 1 on the device path");
  if (m < 0 || m > INT32_MAX) return fail(PGX_EINVAL, "edge count must be in [0, 2^31)");
  if (!row_ptr || !graph_ws || (m > 0 && !col_idx))
    return fail(PGX_EINVAL, "null graph pointer");
  return PGX_OK;
}

}  // namespace

// ==================================================================
// C ABI
// ==================================================================

extern "C" {

int pgx_abi_version(void) { return PGX_ABI_VERSION; }

const char *pgx_last_error(void) { return g_last_error.c_str(); }

#ifdef PGX_COUNT_OPS
extern "C" int pgx_debug_counts(unsigned long long *out3) {
  cudaMemcpyFromSymbol(out3, g_dbg_reds, 8, 0);
  cudaMemcpyFromSymbol(out3 + 1, g_dbg_bits, 8, 0);
  cudaMemcpyFromSymbol(out3 + 2, g_dbg_edges, 8, 0);
  unsigned long long z = 0;
  cudaMemcpyToSymbol(g_dbg_reds, &z, 8, 0);
  cudaMemcpyToSymbol(g_dbg_bits, &z, 8, 0);
  cudaMemcpyToSymbol(g_dbg_edges, &z, 8, 0);
  return 0;
}
#endif

int pgx_set_option(int key, int value) {
  if (key < 0 || key >= PGX_OPT_COUNT) return fail(PGX_EINVAL, "unknown option");
  g_opt[key] = value;
  return PGX_OK;
}

int pgx_device_sm_count(int device, int *sm_count) {
  if (!sm_count) return fail(PGX_EINVAL, "null out pointer");
  PGX_CUDA(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, device));
  return PGX_OK;
}

int pgx_offsets_to_i32(const int64_t *offsets64, int32_t *row_ptr, int64_t count,
                       uintptr_t stream) {
  if (count < 0 || (count && (!offsets64 || !row_ptr))) return fail(PGX_EINVAL, "bad offsets");
  if (!count) return PGX_OK;
  const int grid = (int)std::min<int64_t>(ceil_div(count, 256), 148 * 16);
  offsets_to_i32_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(offsets64, row_ptr, count);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_graph_workspace_bytes(int64_t n, int64_t m, size_t *bytes) {
  if (!bytes || n < 0 || m < 0) return fail(PGX_EINVAL, "bad sizes");
  *bytes = graph_ws_layout(n, m, nullptr, nullptr);
  return PGX_OK;
}

int pgx_graph_prepare(int32_t n, int64_t m, const int32_t *row_ptr, void *graph_ws,
                      size_t graph_ws_bytes, uintptr_t stream) {
  if (n < 1 || m < 0 || m > INT32_MAX || !row_ptr || !graph_ws)
    return fail(PGX_EINVAL, "bad graph_prepare arguments");
  GraphWs g;
  if (graph_ws_layout(n, m, &g, (char *)graph_ws) > graph_ws_bytes)
    return fail(PGX_ENOMEM, "graph workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = (int)ceil_div(n, kCompactBlock);
  nz_count_kernel<<<nb, kCompactBlock, 0, st>>>(row_ptr, n, g.blk);
  nz_scan_blocks_kernel<<<1, kCompactBlock, 0, st>>>(g.blk, nb, g.hdr);
  nz_write_kernel<<<nb, kCompactBlock, 0, st>>>(row_ptr, n, g.blk, g.nz_id, g.nz_eb, m);
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  tile_map_kernel<<<sms * 8, 256, 0, st>>>(g.hdr, g.nz_eb, g.tile_src);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_run_workspace_bytes(int app, int64_t n, int64_t m, int32_t max_supersteps,
                            size_t *bytes) {
  if (!bytes || n < 0 || m < 0 || max_supersteps < 1 || app < 0 || app > 3)
    return fail(PGX_EINVAL, "bad run workspace arguments");
  *bytes = run_ws_layout(app, n, m, max_supersteps, nullptr, nullptr);
  return PGX_OK;
}

static int min_run(int app, int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
                   const void *graph_ws, const int32_t *hub_ids, int32_t nhubs,
                   int32_t source, int32_t max_supersteps, uint32_t *val,
                   void *run_ws, size_t run_ws_bytes, int64_t *stats, uintptr_t stream) {
  if (nhubs < 0 || nhubs > kHubs || (nhubs > 0 && !hub_ids))
    return fail(PGX_EINVAL, "hub count must be in [0, pgx_hub_capacity()]");
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
  if (run_ws_layout(app, n, m, max_supersteps, &p.ws, (char *)run_ws) > run_ws_bytes)
    return fail(PGX_ENOMEM, "run workspace too small");
  p.val = val;
  p.source = source;
  p.max_steps = max_supersteps;
  p.read_filter = g_opt[PGX_OPT_READ_FILTER];
  p.hub_ids = hub_ids;
  p.nhubs = nhubs;
  p.stats = stats;
  cudaStream_t st = (cudaStream_t)stream;
  PGX_CUDA(cudaMemsetAsync(p.ws.bar, 0, 64, st));
  const size_t smem = scatter_smem(PGX_OP_MIN_U32, nhubs);
  int grid = 0;
  void *args[] = {&p};
  if (app == PGX_APP_SSSP) {
    rc = coop_grid(min_run_kernel<PGX_APP_SSSP>, smem, &grid);
    if (rc) return rc;
    PGX_CUDA(cudaLaunchCooperativeKernel((void *)min_run_kernel<PGX_APP_SSSP>, grid, kBlock,
                                         args, smem, st));
  } else {
    rc = coop_grid(min_run_kernel<PGX_APP_CC>, smem, &grid);
    if (rc) return rc;
    PGX_CUDA(cudaLaunchCooperativeKernel((void *)min_run_kernel<PGX_APP_CC>, grid, kBlock,
                                         args, smem, st));
  }
  return PGX_OK;
}

int pgx_sssp_run(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
                 const void *graph_ws, const int32_t *hub_ids, int32_t nhubs, int32_t source,
                 int32_t max_supersteps, uint32_t *dist, void *run_ws, size_t run_ws_bytes,
                 int64_t *stats, uintptr_t stream) {
  return min_run(PGX_APP_SSSP, n, m, row_ptr, col_idx, graph_ws, hub_ids, nhubs, source,
                 max_supersteps, dist, run_ws, run_ws_bytes, stats, stream);
}

int pgx_cc_run(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
               const void *graph_ws, const int32_t *hub_ids, int32_t nhubs,
               int32_t max_supersteps, uint32_t *labels, void *run_ws, size_t run_ws_bytes,
               int64_t *stats, uintptr_t stream) {
  return min_run(PGX_APP_CC, n, m, row_ptr, col_idx, graph_ws, hub_ids, nhubs, 0,
                 max_supersteps, labels, run_ws, run_ws_bytes, stats, stream);
}

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

int pgx_pagerank_pull_run(int32_t n, int64_t m, const int32_t *row_ptr,
                          const int32_t *in_row_ptr, const int32_t *in_col,
                          const void *in_graph_ws, int32_t iterations, double damping,
                          double base, double r0, int32_t max_supersteps, double *rank,
                          void *run_ws, size_t run_ws_bytes, int64_t *stats, uintptr_t stream) {
  int rc = check_graph(n, m, in_row_ptr, in_col, in_graph_ws);
  if (rc) return rc;
  if (!row_ptr) return fail(PGX_EINVAL, "null out-CSR offsets");
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
  cudaStream_t st = (cudaStream_t)stream;
  PGX_CUDA(cudaMemsetAsync(p.ws.bar, 0, 64, st));
  PGX_CUDA(cudaMemsetAsync(p.ws.misc, 0, 64, st));
  const size_t smem = (size_t)kWarps * kSlots * 8 + 16;
  int grid = 0;
  rc = coop_grid(pagerank_pull_kernel, smem, &grid);
  if (rc) return rc;
  void *args[] = {&p};
  PGX_CUDA(cudaLaunchCooperativeKernel((void *)pagerank_pull_kernel, grid, kBlock, args, smem, st));
  return PGX_OK;
}

int pgx_slice_init(int app, int32_t len, int32_t lo, void *val, const int32_t *row_ptr,
                   double *share, double r0, uintptr_t stream) {
  if (len < 0 || !val || (app == PGX_APP_PAGERANK && (!row_ptr || !share)))
    return fail(PGX_EINVAL, "bad slice_init arguments");
  if (!len) return PGX_OK;
  const int grid = (int)std::min<int64_t>(ceil_div(len, 256), 148 * 16);
  slice_init_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      app, len, lo, (uint32_t *)val, row_ptr, (double *)val, share, r0);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_scatter(int op, int dense, const int32_t *col_idx, const int32_t *src_eb,
                const int32_t *src_rs, const int32_t *src_ids, int32_t id_offset,
                const void *src_msg, const int32_t *tile_src, int32_t nsrc, int64_t edges,
                void *mailbox, uint32_t *has_bits, uintptr_t stream) {
  if (op != PGX_OP_MIN_U32 && op != PGX_OP_SUM_F64) return fail(PGX_EINVAL, "unknown op");
  if (edges < 0 || edges > INT32_MAX || nsrc < 0) return fail(PGX_EINVAL, "bad sizes");
  if (edges == 0) return PGX_OK;
  if (!col_idx || !src_eb || !tile_src || !mailbox || (!dense && (!src_rs || !src_msg)) ||
      (dense && !src_ids) || (op == PGX_OP_SUM_F64 && !src_msg))
    return fail(PGX_EINVAL, "null scatter pointer");
  ScatterArgs a;
  a.col = col_idx;
  a.eb = src_eb;
  a.rs = src_rs;
  a.ids = src_ids;
  a.msg = src_msg;
  a.tile_src = tile_src;
  a.nsrc = nsrc;
  a.E = edges;
  a.mailbox = mailbox;
  a.has = has_bits;
  a.id_offset = id_offset;
  a.hub_ids = nullptr;
  a.nhubs = 0;
  const int64_t tiles = ceil_div(edges, kTile);
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(tiles, kWarps),
                                                               (int64_t)sms * PGX_SCATTER_MIN_BLOCKS));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = scatter_smem(op);
  const int rf = g_opt[PGX_OPT_READ_FILTER];
  if (op == PGX_OP_MIN_U32 && !dense) {
    PGX_CUDA(cudaFuncSetAttribute(scatter_kernel<PGX_OP_MIN_U32, MsgSrc::kFrontier>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    scatter_kernel<PGX_OP_MIN_U32, MsgSrc::kFrontier><<<grid, kBlock, smem, st>>>(a, rf);
  } else if (op == PGX_OP_MIN_U32) {
    PGX_CUDA(cudaFuncSetAttribute(scatter_kernel<PGX_OP_MIN_U32, MsgSrc::kSourceId>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    scatter_kernel<PGX_OP_MIN_U32, MsgSrc::kSourceId><<<grid, kBlock, smem, st>>>(a, rf);
  } else if (dense) {
    PGX_CUDA(cudaFuncSetAttribute(scatter_kernel<PGX_OP_SUM_F64, MsgSrc::kShareById>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    scatter_kernel<PGX_OP_SUM_F64, MsgSrc::kShareById><<<grid, kBlock, smem, st>>>(a, rf);
  } else {
    return fail(PGX_EINVAL, "sum scatter needs the dense sender list");
  }
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_slice_counters_bytes(size_t *bytes) {
  if (!bytes) return fail(PGX_EINVAL, "null out pointer");
  *bytes = sizeof(SliceCounters);
  return PGX_OK;
}

int pgx_apply_slice(int app, int32_t len, const int32_t *row_ptr, uint32_t *val,
                    uint32_t *mailbox_slice, int32_t *f_eb, int32_t *f_rs, uint32_t *f_msg,
                    int32_t *tile_src, void *counters, int32_t count_only, uint32_t neutral,
                    uintptr_t stream) {
  if (app != PGX_APP_CC && app != PGX_APP_SSSP) return fail(PGX_EINVAL, "min apps only");
  if (len < 0 || !counters) return fail(PGX_EINVAL, "bad apply_slice arguments");
  if (!len) return PGX_OK;
  const int grid = (int)ceil_div(len, kBlock * 4);
  cudaStream_t st = (cudaStream_t)stream;
  if (app == PGX_APP_CC)
    apply_slice_kernel<PGX_APP_CC><<<grid, kBlock, 0, st>>>(len, row_ptr, val, mailbox_slice, f_eb,
                                                           f_rs, f_msg, tile_src,
                                                           (SliceCounters *)counters, count_only,
                                                           neutral);
  else
    apply_slice_kernel<PGX_APP_SSSP><<<grid, kBlock, 0, st>>>(len, row_ptr, val, mailbox_slice,
                                                             f_eb, f_rs, f_msg, tile_src,
                                                             (SliceCounters *)counters,
                                                             count_only, neutral);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_pr_apply_slice(int32_t len, const int32_t *row_ptr, double *rank, double *mailbox_slice,
                       double *share, double base, double damping, double dangling_over_n,
                       int32_t last, double *partials, uintptr_t stream) {
  if (len < 0 || (len && (!row_ptr || !rank || !mailbox_slice || !share || !partials)))
    return fail(PGX_EINVAL, "bad pr_apply_slice arguments");
  if (!len) return PGX_OK;
  const int grid = (int)ceil_div(len, kBlock);
  pr_apply_slice_kernel<<<grid, kBlock, 0, (cudaStream_t)stream>>>(
      len, row_ptr, rank, mailbox_slice, share, base, damping, dangling_over_n, last, partials);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_rmat_keys(int32_t scale, int64_t first_draw, int64_t num_draws, double a, double b,
                  double c, uint64_t seed, int32_t symmetric, int64_t src_lo, int64_t src_hi,
                  uint64_t *keys, int64_t capacity, int64_t *count, uintptr_t stream) {
  if (scale < 1 || scale > 30 || num_draws < 0 || !keys || !count)
    return fail(PGX_EINVAL, "bad R-MAT arguments");
  if (!num_draws) return PGX_OK;
  const double two53 = 9007199254740992.0;
  const uint64_t ta = (uint64_t)floor(a * two53);
  const uint64_t tab = (uint64_t)floor((a + b) * two53);
  const uint64_t tabc = (uint64_t)floor((a + b + c) * two53);
  uint64_t z = seed + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  const uint64_t base = z ^ (z >> 31);
  const int grid = (int)std::min<int64_t>(ceil_div(num_draws, 256), 148 * 32);
  rmat_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      scale, first_draw, num_draws, ta, tab, tabc, base, symmetric, src_lo, src_hi,
      (unsigned long long *)keys, capacity, (unsigned long long *)count);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

}  // extern "C"
