// pgx_gather.cuh -- K3, PageRank's pull fold (the reference's own PR comm
// mode): every vertex folds its in-neighbours' shares.  Reference:
// _fold_chunk (engine.py:425-457), gather_adjacency (graph.py:380-397).
#pragma once

#include "pgx_common.cuh"

namespace pgx {

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
  int32_t n;                // vertex bound of in_col values (checked builds)
  const double *s_hub;      // HUBS: shared-memory copy of the hub sources' shares
};

// HUBS: in_col holds (0x80000000 | slot) for an edge from hub source
// hub_ids[slot] (the highest out-degree vertices); its share is read from the
// CTA's shared-memory copy s_hub[slot] instead of a scattered global load.
// A warp-wide scattered load costs one L1 tag cycle per distinct line
// (hit or miss), which is what bounds the fold (K3); lanes
// whose source is a hub drop out of it.  Same values, same order: the
// result is bit-identical to the plain fold.
template <bool HUBS = false>
__device__ __forceinline__ void gather_phase(const GatherArgs &a, char *smem) {
  const int lane = (int)lane_id();
  const int warp = threadIdx.x >> 5;
  int32_t *s_eb = reinterpret_cast<int32_t *>(smem) + warp * kSlots;
  int32_t *s_id = reinterpret_cast<int32_t *>(smem) + kWarps * kSlots + warp * kSlots;
  const uint64_t pol = evict_first_policy();
  const int64_t ntiles = (a.E + kTile - 1) / kTile;
#if PGX_DYN_TILES  // the scatter's tile schedule (pgx_scatter.cuh)
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
  for (int64_t t = claim(); t >= 0; t = claim()) {
#else
  const int64_t gwarp = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  for (int64_t t = gwarp; t < ntiles; t += nwarps) {
#endif
    const int64_t e0 = t * kTile;
    const int64_t e1 = min(a.E, e0 + kTile);
    const int i0 = a.tile_src[t];
    const int i1 = (t + 1 < ntiles) ? a.tile_src[t + 1] : a.nsrc - 1;
    const int k = i1 - i0 + 1;
    PGX_ASSERT(i0 >= 0 && k >= 1 && k <= kTile + 1 && i1 < a.nsrc);
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
    const bool full = active && a1 - a0 == 8;
    if (full) {
      ld_stream8(a.in_col + a0, pol, col);
    } else {
#pragma unroll
      for (int j = 0; j < 8; j++) col[j] = (a0 + j < a1) ? ld_stream(a.in_col + a0 + j, pol) : 0;
    }
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const bool valid = full || a0 + j < a1;
      if (HUBS) {
        PGX_ASSERT(col[j] < a.n);
        x[j] = !valid ? 0.0 : (col[j] < 0) ? a.s_hub[col[j] & 0x7FFFFFFF] : __ldg(a.share + col[j]);
      } else {
        PGX_ASSERT(col[j] >= 0 && col[j] < a.n);
        x[j] = valid ? __ldg(a.share + col[j]) : 0.0;
      }
    }
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


// A tile-spanning row's fold: tail[t0] + head[t0 + 1] + ... + head[t1], in
// tile order (deterministic).  The loads are issued kSpanBatch at a time
// ahead of the ordered adds: a hub row spans many tiles (C4's largest
// ~70) and one dependent load per tile was the compute phase's critical
// path.
#ifndef PGX_SPAN_BATCH
#define PGX_SPAN_BATCH 16
#endif
constexpr int kSpanBatch = PGX_SPAN_BATCH;

__device__ __forceinline__ double span_sum(const double *head, const double *tail, int64_t t0,
                                           int64_t t1) {
  double f = tail[t0];
  int64_t t = t0 + 1;
  for (; t + kSpanBatch <= t1 + 1; t += kSpanBatch) {
    double h[kSpanBatch];
#pragma unroll
    for (int j = 0; j < kSpanBatch; j++) h[j] = head[t + j];
#pragma unroll
    for (int j = 0; j < kSpanBatch; j++) f = __dadd_rn(f, h[j]);
  }
  for (; t <= t1; t++) f = __dadd_rn(f, head[t]);
  return f;
}

}  // namespace pgx
