// pgx_common.cuh -- shared constants, device helpers, grid barrier and
// workspace layouts of libpgx (B200 / sm_100a).  Included by every
// translation unit; all device code lives in headers so each .cu compiles
// stand-alone (no relocatable device code).
#pragma once

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
#define PGX_MIN_BLOCKS 1     // persistent CTAs of 1024 threads per SM (64 regs)
#endif
#ifndef PGX_PREFETCH
#define PGX_PREFETCH 1       // dense scatter: L2 bulk prefetch of the next tile's ids
#endif
#ifndef PGX_DYN_TILES
#define PGX_DYN_TILES 1      // warps claim tiles from a per-CTA counter (strided tiles)
#endif
#ifndef PGX_PASS
#define PGX_PASS 4           // 32-edge rounds in flight per scatter pass
#endif

// Checked build (-DPGX_DEBUG_CHECKS=1): every index the hot phases compute
// is bounds-checked on the device; a violation prints and traps (the run
// fails with a CUDA error).  compute-sanitizer is not available on the
// test pool, so the GPU suite runs against this build instead.
#ifndef PGX_DEBUG_CHECKS
#define PGX_DEBUG_CHECKS 0
#endif
#define PGX_ASSERT(c)                                                      \
  do {                                                                     \
    if (PGX_DEBUG_CHECKS && !(c)) {                                        \
      printf("PGX_ASSERT failed %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      __trap();                                                            \
    }                                                                      \
  } while (0)

namespace pgx {

// One 1024-thread CTA per SM (measured against 2 x 512: C2 -4 %, C3 -5 %,
// C4 -2 %, C5 -5 %; half the CTAs at every grid barrier, and one shared
// segment twice as large for the segmented scatter)
#ifndef PGX_BLOCK
#define PGX_BLOCK 1024
#endif
constexpr int kBlock = PGX_BLOCK;    // threads per CTA
constexpr int kWarps = kBlock / 32;
constexpr int kItems = 8;            // 32-edge rounds per warp tile
constexpr int kTile = 32 * kItems;   // 256 edges per warp tile
constexpr int kPass = PGX_PASS;
constexpr int kSlots = kTile + 2;    // sources per warp tile (+ sentinel)
constexpr uint32_t kNeutralMin = 0xFFFFFFFFu;
constexpr int kHubs = 12288;         // hub recipients cached per CTA (48 KB smem)
constexpr int kInvalidEdge = 0x7FFFFFFF;  // never a vertex id (n < 2^31 - 1)
#ifndef PGX_APPLY_LIST
#define PGX_APPLY_LIST 24576
#endif
// apply: vertex-id list segment, inside the scatter windows (99 KB); 24576
// entries hold a dense C5 chunk (~15 K recipients) in one segment (C5
// -0.3 %, C2 -0.5 % vs 12288, profiles/ab_r2_apply_list.log)
constexpr int kApplyListBytes = PGX_APPLY_LIST * 4;
static_assert(kApplyListBytes <= kWarps * kSlots * 12, "the list lives in the scatter windows");
constexpr int kMaxCtas = 4096;
// pull PageRank: hub sources whose shares each CTA keeps in shared memory.
// With the fold's per-warp staging (kWarps * kSlots * 8 = 66 KB) a 96 KB
// table takes the 164 KB shared-memory carveout and leaves 92 KB of L1,
// which the fold's scattered loads need in flight: C4 5.76 ms (no table),
// 5.33 (6K), 5.29 (12K), 5.59 (14K, 60 KB of L1), 9.33 (20K, 28 KB of L1)
// (tools/pr_hub_probe.py, DESIGN.md 3 K3)
constexpr int kPrHubCap = 12288;
constexpr int kCompactBlock = 1024;

// ---- host-side error state and knobs (defined in pgx_graph.cu) ----------
extern thread_local std::string g_last_error;
extern int g_opt[PGX_OPT_COUNT];

inline int fail(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}

inline int cuda_fail(cudaError_t e, const char *what) {
  return fail(PGX_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define PGX_CUDA(call)                                       \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) return ::pgx::cuda_fail(_e, #call); \
  } while (0)

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

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

// Vertex slot v of a state array: S = 0 externalised SoA, S = 1 the
// interleaved {mailbox, value} record array (PGX_LAYOUT_INTERLEAVED).
template <int S, typename T>
__device__ __forceinline__ T *slot(T *base, int64_t v) {
  return base + (v << S);
}

__device__ __forceinline__ void red_min_u32(uint32_t *p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.min.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// system scope: slots other GPUs combine into as well (the fused peer
// exchange); a .gpu-scoped atomic is not atomic against another device's
__device__ __forceinline__ void red_min_u32_sys(uint32_t *p, uint32_t v) {
  asm volatile("red.relaxed.sys.global.min.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void red_or_b32_sys(uint32_t *p, uint32_t v) {
  asm volatile("red.relaxed.sys.global.or.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void red_or_b32(uint32_t *p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ __attribute__((unused)) unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Grid barrier for a co-resident (cooperative) grid.  After the barrier
// the weak, L1-cacheable mailbox / has-bit reads of the next phase must not
// see values from before it: the acquire poll invalidates L1 (CCTL.IVALL
// in the SASS), and the release add orders the CTA's writes (bar.sync,
// then MEMBAR.ALL.GPU + RED by thread 0; PTX release is cumulative over
// what happens-before it through the bar.sync).
struct GridBarrier {
  unsigned count;
  unsigned gen;
};

// Two arrival schemes:
//   kArriveRed (every kernel): a monotonic arrival counter (zeroed before
//     every launch); every CTA arrives with one fire-and-forget
//     red.release and polls with ld.acquire until the whole generation
//     arrived -- no atomic return value and no last-arriver hop on the
//     critical path.  1.30 us per barrier at 148 CTAs, 1.54 us with the
//     sequentially consistent fences of PGX_BAR_SC = 1 (MEMBAR.SC.GPU on
//     both sides), 2.06 us for kArriveAtomic (tools/barrier_bench.cu);
//     C1 -14 %, C3 -4 %, C2 -1.4 %, C4 -0.6 % against the fenced version;
//   kArriveAtomic: atomicAdd with return, the last arriver flips `gen`
//     (kept for A/B builds: -DPGX_BAR_DEFAULT=kArriveAtomic).
enum BarrierKind { kArriveAtomic = 0, kArriveRed = 1 };

#ifndef PGX_BAR_SC
#define PGX_BAR_SC 0       // 1: sequentially consistent fences around the red arrival
#endif
#ifndef PGX_BAR_DEFAULT
#define PGX_BAR_DEFAULT kArriveRed
#endif
template <int KIND = PGX_BAR_DEFAULT>
__device__ __forceinline__ void grid_sync(GridBarrier *bar, unsigned &gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (KIND != kArriveRed || PGX_BAR_SC) __threadfence();
    if (KIND == kArriveRed) {
      const unsigned target = (gen + 1) * gridDim.x;
      asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(&bar->count), "r"(1u)
                   : "memory");
      // wrap-safe: the counter is monotonic within a launch and may pass
      // 2^32 on very long runs; compare the signed distance
      while ((int)(ld_acquire(&bar->count) - target) < 0) {
      }
    } else {
      const unsigned arrived = atomicAdd(&bar->count, 1u);
      if (arrived == gridDim.x - 1) {
        bar->count = 0;
        __threadfence();
        atomicExch(&bar->gen, gen + 1);
      } else {
        while (ld_acquire(&bar->gen) == gen) {
        }
      }
    }
    // without PGX_BAR_SC the red barrier's release add (MEMBAR.ALL.GPU +
    // RED) and acquire poll (which invalidates L1: CCTL.IVALL) carry the
    // ordering
    if (KIND != kArriveRed || PGX_BAR_SC) __threadfence();
  }
  gen += 1;
  __syncthreads();
}

// kArriveRed grid barrier that also hands the CTA up to two 64-bit
// counters written before it: thread 0 reads them once after the barrier
// and the closing __syncthreads publishes them in shared memory.  Every
// thread loading a counter itself right after a barrier (L1 invalidated)
// sends ~4.7k requests to one L2 line (C3: 30 % of the warp stall samples
// of the unit-weight SSSP kernel, ncu source view).
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_sync_bc(GridBarrier *bar, unsigned &gen,
                                             const unsigned long long *a,
                                             const unsigned long long *b,
                                             unsigned long long *s_out) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (PGX_BAR_SC) __threadfence();
    const unsigned target = (gen + 1) * gridDim.x;
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(&bar->count), "r"(1u)
                 : "memory");
    while ((int)(ld_acquire(&bar->count) - target) < 0) {
    }
    if (PGX_BAR_SC) __threadfence();
    if (a) s_out[0] = ld_relaxed_u64(a);
    if (b) s_out[1] = ld_relaxed_u64(b);
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

inline size_t graph_ws_layout(int64_t n, int64_t m, GraphWs *ws, char *base) {
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
  double *hub_share[2];    // pull PR: [kPrHubCap] x 2 hub sources' shares (by slot)
  uint32_t *snd[2];        // [n/32+2] x 2 senders bitmaps (segmented scatter; min apps)
  uint32_t *sv[2];         // CC: [n] x 2 send values (the neutral for non-senders)
};

inline size_t run_ws_layout(int app, int64_t n, int64_t m, int32_t max_steps, RunWs *ws,
                     char *base, bool interleaved = false) {
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
  // interleaved layout (min programs): {mailbox, value} records
  w.mailbox = take(W * (size_t)(n + 1) * (interleaved && !pr ? 2 : 1));
  w.share2 = w.head = w.tail = nullptr;
  w.hub_share[0] = w.hub_share[1] = nullptr;
  w.snd[0] = w.snd[1] = nullptr;
  w.sv[0] = w.sv[1] = nullptr;
  if (app == PGX_APP_PAGERANK_PULL) {
    w.share2 = (double *)take(sizeof(double) * (size_t)(n + 1));
    w.head = (double *)take(sizeof(double) * (size_t)(ceil_div(m, kTile) + 2));
    w.tail = (double *)take(sizeof(double) * (size_t)(ceil_div(m, kTile) + 2));
    w.hub_share[0] = (double *)take(sizeof(double) * (size_t)kPrHubCap);
    w.hub_share[1] = (double *)take(sizeof(double) * (size_t)kPrHubCap);
  }
  if (!pr) {
    w.f_eb = (int32_t *)take(sizeof(int32_t) * (size_t)(n + 1));
    w.f_rs = (int32_t *)take(sizeof(int32_t) * (size_t)(n + 1));
    w.has = (uint32_t *)take(sizeof(uint32_t) * (size_t)(n / 32 + 2));
    w.tile_src = (int32_t *)take(sizeof(int32_t) * (size_t)(ceil_div(m, kTile) + 2));
    w.snd[0] = (uint32_t *)take(sizeof(uint32_t) * (size_t)(n / 32 + 2));
    w.snd[1] = (uint32_t *)take(sizeof(uint32_t) * (size_t)(n / 32 + 2));
    {  // CC and unit-weight SSSP
      w.sv[0] = (uint32_t *)take(sizeof(uint32_t) * (size_t)(n + 4));  // whole uint4 stores
      w.sv[1] = (uint32_t *)take(sizeof(uint32_t) * (size_t)(n + 4));
    }
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
  int32_t cas_loop;       // ablation: CAS retry loop instead of red.min
  uint32_t neutral;       // min neutral of the mailbox (has-bit publication)
  int32_t n;              // vertex bound of col_idx values (checked builds)
  // fused peer-memory exchange (pgx_scatter_peer): a message that passes
  // the local filter and whose recipient another rank owns is also
  // combined into the owner's mailbox, peer_mb[owner] (NVLink P2P)
  uint32_t *const *peer_mb;  // [world] mailbox base of every rank
  const int32_t *bounds;     // [world + 1] owner ranges
  int32_t world;
  int32_t lo, hi;            // this rank's own range
};

// shared memory of the scatter: one source window per warp (+ the hub
// cache of the min combiner, right after the windows)
__host__ __device__ constexpr size_t scatter_windows_smem(int op) {
  // s_eb (4 B) + {message | row offset, message} (8 B) per slot; the apply
  // reuses the same region for its recipient list
  return (size_t)kWarps * kSlots * (sizeof(int32_t) + 8) > (size_t)kApplyListBytes
             ? (size_t)kWarps * kSlots * (sizeof(int32_t) + 8)
             : (size_t)kApplyListBytes;
}
__host__ __device__ constexpr size_t scatter_smem(int op, int nhubs = 0) {
  return scatter_windows_smem(op) + (op == PGX_OP_MIN_U32 ? sizeof(uint32_t) * nhubs : 0) + 16;
}


// block-wide exclusive scan of an int (any multiple-of-32 block size)
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

// launch helper for the persistent (cooperative) kernels: CTAs per SM from
// the occupancy calculator, capped by PGX_OPT_CTAS_PER_SM and kMaxCtas
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

inline int check_graph(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
                       const void *graph_ws) {
  if (n < 1) return fail(PGX_EINVAL, "vertex count must be >= 1 on the device path");
  if (m < 0 || m > INT32_MAX) return fail(PGX_EINVAL, "edge count must be in [0, 2^31)");
  if (!row_ptr || !graph_ws || (m > 0 && !col_idx))
    return fail(PGX_EINVAL, "null graph pointer");
  return PGX_OK;
}

}  // namespace pgx
