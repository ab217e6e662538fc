// pgx_pull.cuh -- K1p, the bottom-up (pull) superstep of unit-weight SSSP.
//
// Unit-weight SSSP sends one uniform message per superstep (the superstep
// index + 1), so the superstep's whole result is the has-message bitmask:
// vertex v receives a message iff one of its in-neighbours is a sender
// (engine.py:154-162 run over every sender's out-edges; the next frontier is
// every vertex holding a pending message, engine.py:349-355, whether or not
// the message improves it).  That set can be computed from the receiving
// side: v scans its in-edges and stops at the first sender -- on a
// superstep whose senders hold a large share of the edges, a couple of
// in-edge checks per vertex instead of one filter read per out-edge
// (direction-optimising BFS).  Bit-identical by construction: the bitmask,
// hence recipients, values and every statistic (the edge / sender counts of
// the superstep come from the apply that built the senders, as for K1).
//
// Three phases, separated by grid barriers (the caller's):
//   A  senders bitmap: bit u = (dist[u] == level), 8 vertices per lane --
//      the senders of superstep s are exactly the vertices whose distance
//      became s in the previous apply;
//   B  one lane per vertex, up to kPullRounds rounds of two in-row sources
//      tested against the bitmap (early exit); a ballot gives the has-word
//      of 32 vertices, stored whole (the bitmask is clear after the
//      previous apply).  A vertex with more in-edges and no sender among
//      the probed ones joins the remainder list: (edge prefix, in-row
//      position, vertex), reserved with one packed 64-bit atomic per warp
//      (the apply's frontier build format, written into the frontier
//      buffers, which a pull superstep does not read);
//   C  the remainders' edges, split into 256-edge warp tiles of that edge
//      space (exact balance: a hub's long in-row spans many tiles); a hit
//      sets the vertex's bit with one red.or per vertex and round.
// Algorithmic traffic (K1p): 4 B distance + 8 B offsets per
// vertex, the probed in-row sources (one or two 32-byte sectors per
// vertex), n/8 B of bitmask; the bitmap tests are L1 requests into a
// 512 KB bitmap (C3).  Measured (C3, B200): superstep 1 63 us vs 152 us
// pushed, superstep 2 94 us vs 134 us.
#pragma once

#include "pgx_common.cuh"

namespace pgx {

#ifndef PGX_PULL_ROUNDS
#define PGX_PULL_ROUNDS 3
#endif
#ifndef PGX_PULL_GROUPS
#define PGX_PULL_GROUPS 2
#endif
constexpr int kPullRounds = PGX_PULL_ROUNDS;  // probe rounds (2 sources each) before deferring
constexpr int kPullGroups = PGX_PULL_GROUPS;  // 32-vertex groups a warp probes at once

struct PullArgs {
  const int32_t *in_row_ptr;  // in-CSR offsets [n+1]
  const int32_t *in_col;      // in-CSR sources, ascending per row
  const uint32_t *dist;       // SSSP distances (the value array)
  int32_t n;
  int64_t m;
  uint32_t level;             // senders hold dist == level
  uint32_t *snd;              // [n/32+2] senders bitmap (scratch)
  uint32_t *has;              // has-message bitmask (clear on entry)
  int32_t *q_eb;              // remainder list: exclusive edge prefix
  int32_t *q_rs;              //   in-row position of the first unprobed edge
  uint32_t *q_v;              //   vertex
  int32_t *q_tile;            //   remainder entry holding each tile's first edge
  unsigned long long *q_ctr;  // entries << 32 | edges (zeroed in phase A)
};

__device__ __forceinline__ bool bit_set(const uint32_t *bm, uint32_t u) {
  return (bm[u >> 5] >> (u & 31u)) & 1u;
}

// phase A: a lane reads 8 consecutive distances (two 16-byte loads), so a
// warp covers 256 vertices = 8 bitmap words per pass and the pass is a few
// independent loads per thread instead of a latency-bound chain
__device__ __forceinline__ void pull_senders_phase(const PullArgs &a) {
  const unsigned nthreads = gridDim.x * blockDim.x;
  const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned lane = lane_id();
  if (gtid == 0) *a.q_ctr = 0ull;
  const bool vec = (reinterpret_cast<uintptr_t>(a.dist) & 15u) == 0;
  for (unsigned v0 = (gtid & ~31u) * 8u; v0 < (unsigned)a.n; v0 += nthreads * 8u) {  // warp-uniform
    const unsigned v = v0 + lane * 8u;
    unsigned bits = 0;
    if (vec && v + 8u <= (unsigned)a.n) {
      const uint4 x = *reinterpret_cast<const uint4 *>(a.dist + v);
      const uint4 y = *reinterpret_cast<const uint4 *>(a.dist + v + 4);
      bits = (x.x == a.level) | (x.y == a.level) << 1 | (x.z == a.level) << 2 |
             (x.w == a.level) << 3 | (y.x == a.level) << 4 | (y.y == a.level) << 5 |
             (y.z == a.level) << 6 | (y.w == a.level) << 7;
    } else {
      for (unsigned k = 0; k < 8u; k++)
        if (v + k < (unsigned)a.n && a.dist[v + k] == a.level) bits |= 1u << k;
    }
    // lanes 4i..4i+3 hold the 4 bytes of word (v0 / 32 + i)
    unsigned w = bits << (8u * (lane & 3u));
    w |= __shfl_down_sync(0xFFFFFFFFu, w, 1);
    w |= __shfl_down_sync(0xFFFFFFFFu, w, 2);
    if ((lane & 3u) == 0 && v < (unsigned)a.n) a.snd[v >> 5] = w;
  }
}

// inclusive warp scan of a u64
__device__ __forceinline__ unsigned long long warp_incl_scan_u64(unsigned long long x) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if ((int)lane_id() >= o) x += y;
  }
  return x;
}

// phase B: warp-synchronous (no block barriers); a warp probes kPullGroups
// groups of 32 consecutive vertices at once, lane j of group g holding
// vertex 32 g + j.  A round tests two in-row sources per lane against the
// bitmap.  The warp's first groups test one source at each end of the row
// in round 0 and learn which end holds the superstep's senders (until one
// end leads by 16 hits; on R-MAT the senders of an early superstep are the
// low-id hubs at the rows' fronts, those of a later one high-id vertices
// at their backs -- C3: 84 % of superstep 1's recipients hit on the first
// source, 70 % of superstep 2's on the last); later groups read the
// preferred end, then the other,
// then the preferred again: one in-row sector per round.  Rounds are few
// (kPullRounds): what they leave unprobed goes to the edge-parallel phase
// C instead of lengthening every warp's dependent chain.  A round runs
// while any lane of the warp needs it.
__device__ __forceinline__ void pull_probe_phase(const PullArgs &a) {
  constexpr int U = kPullGroups, K = kPullRounds;
  const int lane = (int)lane_id();
  const int ngroups = (a.n + 31) >> 5;
  const int gw = blockIdx.x * kWarps + (int)(threadIdx.x >> 5);
  const int nw = gridDim.x * kWarps;
  int score = 0;  // warp-uniform: first-round hits at the back minus at the front
  // groups in descending id order: the low-id hubs, whose long in-rows
  // depend most on the end chosen, come last, after the warp has learnt
  // the superstep's end from many ordinary rows
  const int iters = (ngroups + nw * U - 1) / (nw * U);
  for (int it = iters - 1; it >= 0; it--) {  // warp-uniform
    const int g0 = (it * nw + gw) * U;
    int lo[U], hi[U];  // the unprobed part [lo, hi) of each lane's in-row
    bool hit[U];
    if (g0 >= ngroups) continue;
#pragma unroll
    for (int j = 0; j < U; j++) {
      const int v = ((g0 + j) << 5) + lane;
      lo[j] = hi[j] = 0;
      if (v < a.n) {
        lo[j] = a.in_row_ptr[v];
        hi[j] = a.in_row_ptr[v + 1];
      }
      hit[j] = false;
    }
    const bool learn = score < 16 && score > -16;  // until one end leads clearly
    const bool pref = score > 0;                    // true: the back
    int d_score = 0;
#pragma unroll 1
    for (int k = 0; k < K; k++) {
      bool need = false;
#pragma unroll
      for (int j = 0; j < U; j++) need |= !hit[j] && lo[j] < hi[j];
      if (!__any_sync(0xFFFFFFFFu, need)) break;
      const bool both = learn && k == 0;
      const bool back = (k == 1 && !learn) ? !pref : pref;
      int u0[U], u1[U];
#pragma unroll
      for (int j = 0; j < U; j++) {
        u0[j] = u1[j] = -1;
        if (!hit[j] && lo[j] < hi[j]) {
          if (both) {  // front, back
            u0[j] = __ldg(a.in_col + lo[j]++);
            if (lo[j] < hi[j]) u1[j] = __ldg(a.in_col + --hi[j]);
          } else if (back) {
            u0[j] = __ldg(a.in_col + --hi[j]);
            if (lo[j] < hi[j]) u1[j] = __ldg(a.in_col + --hi[j]);
          } else {
            u0[j] = __ldg(a.in_col + lo[j]++);
            if (lo[j] < hi[j]) u1[j] = __ldg(a.in_col + lo[j]++);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < U; j++) {
        const bool h0 = u0[j] >= 0 && bit_set(a.snd, (uint32_t)u0[j]);
        const bool h1 = u1[j] >= 0 && bit_set(a.snd, (uint32_t)u1[j]);
        hit[j] |= h0 || h1;
        if (both)
          d_score += __popc(__ballot_sync(0xFFFFFFFFu, h1 && !h0)) -
                     __popc(__ballot_sync(0xFFFFFFFFu, h0 && !h1));
      }
    }
    score += d_score;
    unsigned long long mine[U], tot = 0;
#pragma unroll
    for (int j = 0; j < U; j++) {
      const unsigned w = __ballot_sync(0xFFFFFFFFu, hit[j]);
      if (lane == 0 && w) a.has[g0 + j] = w;  // the bitmask is clear: plain store
      const int rem = hit[j] ? 0 : hi[j] - lo[j];
      const unsigned long long x = rem ? ((1ull << 32) | (unsigned long long)rem) : 0ull;
      const unsigned long long incl = warp_incl_scan_u64(x);
      mine[j] = tot + incl - x;  // exclusive, across the warp's groups
      tot += __shfl_sync(0xFFFFFFFFu, incl, 31);
    }
    if (tot == 0) continue;  // warp-uniform
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(a.q_ctr, tot);
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
#pragma unroll
    for (int j = 0; j < U; j++) {
      const int rem = hit[j] ? 0 : hi[j] - lo[j];
      if (!rem) continue;
      const unsigned long long run = base + mine[j];
      const unsigned pos = (unsigned)(run >> 32);
      const int eb = (int)(run & 0xFFFFFFFFull);
      a.q_eb[pos] = eb;
      a.q_rs[pos] = lo[j];
      a.q_v[pos] = (uint32_t)(((g0 + j) << 5) + lane);
      for (int64_t t = ((int64_t)eb + kTile - 1) / kTile; t * kTile < (int64_t)eb + rem; t++)
        a.q_tile[t] = (int)pos;
    }
  }
}

// phase C: the remainders' edges in 256-edge warp tiles.  The tile's
// entries (<= 257, each holds >= 1 edge) are staged in the warp's
// shared-memory window -- edge prefix, in-row position, vertex -- in one
// coalesced pass; each lane then resolves its 8 edges' entries there
// (ascending) and issues all 8 source loads, then all 8 bitmap tests: two
// dependent round trips per tile.  `q` = entries << 32 | edges (read once
// per CTA, grid_sync_bc).
__device__ __forceinline__ void pull_remainder_phase(const PullArgs &a, unsigned long long q,
                                                     char *smem) {
  const int nq = (int)(q >> 32);
  const int64_t E = (int64_t)(q & 0xFFFFFFFFull);
  if (E == 0) return;
  const int lane = (int)lane_id();
  const int warp = (int)(threadIdx.x >> 5);
  int32_t *w_eb = reinterpret_cast<int32_t *>(smem) + warp * kSlots;
  int2 *w_rv = reinterpret_cast<int2 *>(smem + sizeof(int32_t) * kWarps * kSlots) + warp * kSlots;
  const int64_t ntiles = (E + kTile - 1) / kTile;
  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  for (int64_t t = (int64_t)blockIdx.x * kWarps + warp; t < ntiles; t += nwarps) {
    const int j0 = a.q_tile[t];
    const int64_t tend = min((t + 1) * kTile, E);
    // window slot k = entry j0 + k (edge prefix E past the last entry),
    // staged 32 entries at a time up to the first entry starting at or
    // after the tile's end (usually one pass: one round trip, not nine)
    __syncwarp();
    for (int c = 0; c < kSlots - 1; c += 32) {  // warp-uniform
      const int j = j0 + c + lane;
      const bool in = j < nq;
      int eb = (int)E, rs = 0, v = 0;
      if (in) {
        eb = a.q_eb[j];
        rs = a.q_rs[j];
        v = (int)a.q_v[j];
      }
      if (c + lane < kSlots - 1) {
        w_eb[c + lane] = eb;
        w_rv[c + lane] = make_int2(rs, v);
      }
      if (__ballot_sync(0xFFFFFFFFu, (int64_t)eb < tend) != 0xFFFFFFFFu) break;
    }
    __syncwarp();
    int k = 0;  // this lane's entry (window slot), ascending across rounds
    int u[kItems], v[kItems];
#pragma unroll
    for (int r = 0; r < kItems; r++) {
      const int64_t p = t * kTile + r * 32 + lane;
      u[r] = -1;
      v[r] = 0;
      if (p < tend) {
        while (k + 1 < kSlots - 1 && w_eb[k + 1] <= p) k++;
        const int2 rv = w_rv[k];
        v[r] = rv.y;
        u[r] = __ldg(a.in_col + rv.x + (int)(p - w_eb[k]));
      }
    }
    // a long in-row spans whole rounds: one red.or per vertex and round
    // (the lanes sharing a vertex are contiguous; the lowest one publishes)
#pragma unroll
    for (int r = 0; r < kItems; r++) {
      const bool h = u[r] >= 0 && bit_set(a.snd, (uint32_t)u[r]);
      const unsigned same = __match_any_sync(0xFFFFFFFFu, v[r]);
      const unsigned hits = __ballot_sync(0xFFFFFFFFu, h) & same;
      if (hits && lane == __ffs(same) - 1)
        red_or_b32(a.has + (v[r] >> 5), 1u << (v[r] & 31));
    }
  }
}

}  // namespace pgx
