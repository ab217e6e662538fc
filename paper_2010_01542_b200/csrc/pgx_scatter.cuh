// pgx_scatter.cuh -- K1, the superstep's scatter: every sender pushes its
// message along its out-edges and the messages are combined into each
// recipient's single mailbox slot.  Reference: send_to_out_neighbors
// (engine.py:154-162), send_hybrid / apply_cas (mailbox.py:147-199),
// edge_balanced_partition (scheduler.py:91-116).
#pragma once

#include "pgx_common.cuh"

namespace pgx {

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

// Debug build only (-DPGX_COUNT_OPS=1, tools/count_ops.py): per-TU device
// counters of the scatter's operations -- [0] red.min, [1] has-bit red.or,
// [2] edges -- read and reset by pgx_debug_counts (not part of pgx.h).
#ifndef PGX_COUNT_OPS
#define PGX_COUNT_OPS 0
#endif
#if PGX_COUNT_OPS
static __device__ unsigned long long g_pgx_ops[3];
#define PGX_COUNT(i) (c_ops[i]++)
#else
#define PGX_COUNT(i) ((void)0)
#endif

// BFS = true: unit-weight SSSP, where every message of a superstep has the
// same value (the superstep index + 1), so the min-combined mailbox carries
// no information beyond "received": the filter reads the has-message bit
// (a 512 KB bitmap instead of the 16.8 MB mailbox for C3 -- 1024 vertices
// per line, mostly L1 hits) and a clear bit is set with one red.or.
template <int OP, MsgSrc MS, int S = 0, bool PEER = false, bool BFS = false>
__device__ void scatter_phase(const ScatterArgs &a, char *smem, bool read_filter = true) {
  using Msg = typename std::conditional<OP == PGX_OP_SUM_F64, double, uint32_t>::type;
  constexpr bool kDense = MS != MsgSrc::kFrontier;
  const int lane = (int)lane_id();
  const int warp = threadIdx.x >> 5;
  // per-warp source window: row starts (boundary candidates) and, per
  // source, either the message (dense senders: pos = e) or the packed pair
  // {row offset - edge base, message} (sparse frontier: pos = e + off)
  int32_t *s_eb = reinterpret_cast<int32_t *>(smem) + warp * kSlots;
  char *s_second = smem + sizeof(int32_t) * kWarps * kSlots;
  Msg *s_msg = reinterpret_cast<Msg *>(s_second) + warp * kSlots;
  uint2 *s_om = reinterpret_cast<uint2 *>(s_second) + warp * kSlots;
  const uint64_t pol = evict_first_policy();
  const int64_t ntiles = (a.E + kTile - 1) / kTile;
  const unsigned upto = (lane == 31) ? 0xFFFFFFFFu : ((2u << lane) - 1u);
  uint32_t *s_hub = reinterpret_cast<uint32_t *>(smem + scatter_windows_smem(OP));
#if PGX_COUNT_OPS
  unsigned long long c_ops[3] = {0ull, 0ull, 0ull};
#endif
  if (OP == PGX_OP_MIN_U32 && a.nhubs > 0) {  // block-uniform
    for (int i = threadIdx.x; i < a.nhubs; i += blockDim.x) s_hub[i] = kNeutralMin;
    __syncthreads();
  }

#if PGX_DYN_TILES
  // Tile schedule: CTA b owns tiles b, b + grid, b + 2 grid, ... (spread
  // over the whole edge space, like a static stride) and its warps claim
  // them one at a time from a shared-memory counter (no global atomics), so
  // a slow tile delays only its own warp's next claim, not a fixed share.
  __shared__ unsigned s_tctr;
  if (threadIdx.x == 0) s_tctr = 0u;
  __syncthreads();
  auto claim = [&]() -> int64_t {
    unsigned c = 0u;
    if (lane == 0) c = atomicAdd(&s_tctr, 1u);
    c = __shfl_sync(0xFFFFFFFFu, c, 0);
    const int64_t tt = (int64_t)blockIdx.x + (int64_t)c * gridDim.x;
    return tt < ntiles ? tt : -1;
  };
  int64_t t = claim();
#else
  const int64_t gwarp = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  int64_t t = gwarp < ntiles ? gwarp : -1;
#endif
  while (t >= 0) {
#if PGX_DYN_TILES
    const int64_t tnext = claim();  // one ahead: its ids can be prefetched
#else
    const int64_t tnext = t + nwarps < ntiles ? t + nwarps : -1;
#endif
    const int64_t e0 = t * kTile;
    const int64_t e1 = min(a.E, e0 + kTile);
#if PGX_PREFETCH
    // the warp's next tile: its neighbour ids (dense: one contiguous 1 KB
    // run of col_idx) are pulled into L2 while this tile is processed
    if (kDense && lane == 0 && tnext >= 0) {
      // the bulk prefetch needs 16-byte granules: widen the range (col_idx
      // itself may be any 4-byte-aligned view, e.g. a rank's slice)
      const int64_t en = tnext * kTile;
      const uint64_t p0 = reinterpret_cast<uint64_t>(a.col + en) & ~15ull;
      const uint64_t p1 =
          (reinterpret_cast<uint64_t>(a.col + min(a.E, en + kTile)) + 15ull) & ~15ull;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p0),
                   "r"((unsigned)(p1 - p0))
                   : "memory");
    }
#endif
    const int i0 = a.tile_src[t];
    const int i1 = (t + 1 < ntiles) ? a.tile_src[t + 1] : a.nsrc - 1;
    const int k = i1 - i0 + 1;  // <= kTile + 1
    PGX_ASSERT(i0 >= 0 && k >= 1 && k <= kTile + 1 && i1 < a.nsrc);
    __syncwarp();
    for (int j = lane; j <= k; j += 32) {
      const int i = i0 + j;
      if (j < k) {
        const int32_t eb = a.eb[i];
        s_eb[j] = eb;
        if (MS == MsgSrc::kFrontier) {
          s_om[j] = make_uint2((uint32_t)(a.rs[i] - eb),
                               (uint32_t)reinterpret_cast<const uint32_t *>(a.msg)[i]);
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

    int cur = 0;  // s_eb[0] <= e0: tile_src names the source holding e0
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
          const int64_t pp = (int64_t)s_eb[ci] - base;
          if (pp >= 0 && pp < 32) bit = 1u << pp;
        }
        const unsigned bm = __reduce_or_sync(0xFFFFFFFFu, bit);
        const int src = cur + __popc(bm & upto);
        cur += __popc(bm);
        w[r] = kInvalidEdge;
        if (e < e1) {
          PGX_ASSERT(src >= 0 && src < k);
          int64_t pos = e;
          if (kDense) {
            mv[r] = s_msg[src];
          } else {
            const uint2 om = s_om[src];
            pos = e + (int32_t)om.x;
            mv[r] = (Msg)om.y;
          }
          w[r] = ld_stream(a.col + pos, pol);
          PGX_ASSERT(w[r] < 0 || w[r] < a.n);
        }
      }
      if (OP == PGX_OP_MIN_U32 && BFS) {
        uint32_t hw[kPass];
#pragma unroll
        for (int r = 0; r < kPass; r++) {
          const int x = w[r];
          hw[r] = (x == kInvalidEdge) ? 0xFFFFFFFFu : a.has[x >> 5];
        }
#pragma unroll
        for (int r = 0; r < kPass; r++) {
          const int x = w[r];
          if (x != kInvalidEdge) PGX_COUNT(2);
          if (x != kInvalidEdge && !((hw[r] >> (x & 31)) & 1u)) {
            const uint32_t bit = 1u << (x & 31);
            if (PEER && x >= a.lo && x < a.hi) {
              red_or_b32_sys(a.has + (x >> 5), bit);  // peers set owned bits too
            } else {
              red_or_b32(a.has + (x >> 5), bit);
              if (PEER) {
                // the local bit is this rank's filter; the owner's bit is the
                // exchange (peer_mb = the ranks' has-bitmaps here), over
                // NVLink when the owner is another GPU
                int o = 0;
                while (o + 1 < a.world && x >= __ldg(a.bounds + o + 1)) o++;
                red_or_b32_sys(a.peer_mb[o] + (x >> 5), bit);
              }
            }
            PGX_COUNT(1);
          }
        }
      } else if (OP == PGX_OP_MIN_U32) {
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
                   : (read_filter ? *slot<S>(mb, x) : a.neutral);
        }
#pragma unroll
        for (int r = 0; r < kPass; r++) {
          const int x = w[r];
          const uint32_t msg = (uint32_t)mv[r];
          if (x != kInvalidEdge) PGX_COUNT(2);
          if (x != kInvalidEdge && msg < old[r]) {
            int v = x;
            uint32_t prev = old[r];
            if (x < 0) {  // hub: the CTA-local copy let it through; consult
                          // the global slot (the shared filter) before the red
              const int hs = x & 0x7FFFFFFF;
              v = a.hub_ids[hs];
              prev = *slot<S>(mb, v);
              s_hub[hs] = min(prev, msg);  // racy store: only weakens the filter
              if (msg >= prev) v = -1;
            }
            if (v >= 0) {
              if (a.cas_loop) {  // ablation: lock-style CAS retry per message
                uint32_t cur = prev;
                while (msg < cur) {
                  const uint32_t got = atomicCAS(slot<S>(mb, v), cur, msg);
                  if (got == cur) break;
                  cur = got;
                }
                if (a.has && prev == a.neutral) atomicOr(a.has + (v >> 5), 1u << (v & 31));
              } else {
                // owned slots of a peer-exchange rank are combined into by
                // the other GPUs too: system-scope atomics there
                if (PEER && v >= a.lo && v < a.hi) red_min_u32_sys(slot<S>(mb, v), msg);
                else red_min_u32(slot<S>(mb, v), msg);
                PGX_COUNT(0);
                if (a.has && prev == a.neutral) {
                  red_or_b32(a.has + (v >> 5), 1u << (v & 31));
                  PGX_COUNT(1);
                }
              }
              if (PEER && (v < a.lo || v >= a.hi)) {
                // the local slot is this rank's filter; the owner's slot is
                // the combined mailbox: one more fire-and-forget red.min,
                // over NVLink when the owner is another GPU
                int o = 0;
                while (o + 1 < a.world && v >= __ldg(a.bounds + o + 1)) o++;
                red_min_u32_sys(a.peer_mb[o] + v, msg);
              }
            }
          }
        }
      } else {
        double *mb = reinterpret_cast<double *>(a.mailbox);
#pragma unroll
        for (int r = 0; r < kPass; r++)
          if (w[r] != kInvalidEdge) atomicAdd(mb + w[r], (double)mv[r]);
      }
    }
    t = tnext;
  }
#if PGX_COUNT_OPS
  for (int i = 0; i < 3; i++)
    if (c_ops[i]) atomicAdd(&g_pgx_ops[i], c_ops[i]);
#endif
}


// Ablation arm of the scheduler (harness.py:273-292 grid): one thread per
// sender walks its whole out-row (the reference's vertex-centric split,
// scheduler.py:79-88).  No edge balance: a hub row serialises on one lane.
template <MsgSrc MS, int S = 0>
__device__ void scatter_vertex_phase(const ScatterArgs &a, bool read_filter) {
  constexpr bool kDense = MS != MsgSrc::kFrontier;
  uint32_t *mb = reinterpret_cast<uint32_t *>(a.mailbox);
  const int nthreads = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.nsrc; i += nthreads) {
    const int64_t eb = a.eb[i];
    const int64_t ee = (i + 1 < a.nsrc) ? a.eb[i + 1] : a.E;
    const int64_t rs = kDense ? eb : (int64_t)a.rs[i];
    const uint32_t msg = (MS == MsgSrc::kFrontier)
                             ? reinterpret_cast<const uint32_t *>(a.msg)[i]
                             : (uint32_t)(a.ids[i] + a.id_offset);
    for (int64_t e = eb; e < ee; e++) {
      const int v = a.col[rs + (e - eb)];
      const uint32_t prev = read_filter ? *slot<S>(mb, v) : a.neutral;
      if (msg < prev) {
        if (a.cas_loop) {
          uint32_t cur = prev;
          while (msg < cur) {
            const uint32_t got = atomicCAS(slot<S>(mb, v), cur, msg);
            if (got == cur) break;
            cur = got;
          }
        } else {
          red_min_u32(slot<S>(mb, v), msg);
        }
        if (a.has && prev == a.neutral) red_or_b32(a.has + (v >> 5), 1u << (v & 31));
      }
    }
  }
}

}  // namespace pgx
