// pgx_apply.cuh -- K2, the superstep's apply for the min programs: consume
// the mailbox, compute (adopt an improvement), vote to halt, build the next
// frontier.  Reference: _chunk_push (engine.py:402-414), the computes of
// connected_components / sssp (algorithms.py:99-108, 136-147),
// _next_frontier (engine.py:349-365).
#pragma once

#include "pgx_common.cuh"

namespace pgx {

// ------------------------------------------------------------------
// sparse apply for the min programs (SSSP / CC), driven by the
// has-message bitmask: consume every flagged mailbox (vertex order),
// adopt an improvement, append improved vertices to the next frontier
// with their edge prefix.  One 64-bit atomic per apply batch reserves
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

// Apply chunk: every CTA takes kBlock bitmask words (one per thread, in
// 32-word groups interleaved across the grid; a quiet chunk costs one load
// and one barrier).  The set bits are compacted
// into a shared-memory vertex list (block scan of popcounts, segments of
// kListCap ids), which is consumed in batches of kApplyItems independent
// recipients per thread -- a handful of dependent round trips per chunk
// instead of one serial chain per 64 words.
#ifndef PGX_APPLY_ITEMS
#define PGX_APPLY_ITEMS 4
#endif
constexpr int kApplyItems = PGX_APPLY_ITEMS;
#ifndef PGX_APPLY_PREFETCH
#define PGX_APPLY_PREFETCH 1
#endif
constexpr int kListCap = kApplyListBytes / (int)sizeof(int32_t);

// Returns (recipients counted) << 32 | (broadcasts) for this thread.  With
// `count_only` the bitmask is only counted (superstep cap reached: the
// pending messages must stay unconsumed, engine.py:299-300).
// BFS = true (unit-weight SSSP, see scatter_phase): every flagged recipient
// received the uniform message `bfs_msg`; the mailbox is not used.
template <int APP, int S = 0, bool BFS = false>
__device__ unsigned long long apply_min_phase(const int32_t *__restrict__ row_ptr, uint32_t *val,
                                              uint32_t *mailbox, int32_t n, const RunWs &ws,
                                              StepCounters *ctr, char *smem, bool count_only,
                                              uint32_t bfs_msg = 0, uint32_t *snd = nullptr,
                                              uint32_t *sv = nullptr,
                                              bool no_frontier = false) {
  __shared__ unsigned long long s_w[33];
  __shared__ unsigned long long s_gbase;
  int32_t *s_list = reinterpret_cast<int32_t *>(smem);  // kListCap vertex ids
  uint32_t *f_msg = reinterpret_cast<uint32_t *>(ws.f_msg);
  const int words = (n + 31) >> 5;
  unsigned bcast = 0, recips = 0;
  if (count_only) {
    for (int wi = blockIdx.x * kBlock + threadIdx.x; wi < words; wi += gridDim.x * kBlock)
      recips += __popc(ws.has[wi]);
    return ((unsigned long long)recips << 32);
  }
  // warp w of CTA b takes 32-word group gb + w * grid + b: consecutive
  // groups go to consecutive CTAs, which spreads the dense
  // (low-id) region of a power-law graph over the whole grid
  const int groups = (words + 31) >> 5;
#if PGX_APPLY_PREFETCH
  // the next chunk's word is loaded before this chunk is processed: a
  // quiet chunk then costs a barrier, not a load round trip
  auto load_word = [&](int gb) -> uint32_t {
    const int g = gb + (int)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    const int wi = g * 32 + (int)lane_id();
    return (g < groups && wi < words) ? ws.has[wi] : 0u;
  };
  uint32_t next_word = load_word(0);
#endif
  for (int gb = 0; gb < groups; gb += gridDim.x * kWarps) {  // block-uniform
    const int g = gb + (int)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    const int wi = g * 32 + (int)lane_id();
#if PGX_APPLY_PREFETCH
    const uint32_t word = next_word;
    next_word = load_word(gb + gridDim.x * kWarps);
    if (word) ws.has[wi] = 0u;
#else
    uint32_t word = 0;
    if (g < groups && wi < words) {
      word = ws.has[wi];
      if (word) ws.has[wi] = 0u;
    }
#endif
    if (!__syncthreads_or(word != 0)) continue;  // quiet chunk: one barrier
    const int c = __popc(word);
    recips += c;
    unsigned long long tot64;
    const int off = (int)block_excl_scan_u64((unsigned long long)c, s_w, &tot64);
    const int T = (int)tot64;
    for (int seg = 0; seg < T; seg += kListCap) {  // block-uniform
      // ---- expand this segment of the set bits into s_list (vertex order) ----
      if (off < seg + kListCap && off + c > seg) {
        int o = off;
        uint32_t rem = word;
        while (rem) {
          const int b = __ffs(rem) - 1;
          rem &= rem - 1;
          if (o >= seg && o < seg + kListCap) s_list[o - seg] = (wi << 5) + b;
          o++;
        }
      }
      __syncthreads();
      const int cnt = min(kListCap, T - seg);
      for (int b0 = 0; b0 < cnt; b0 += kBlock * kApplyItems) {  // block-uniform
        // ---- consume + compute, kApplyItems independent recipients / thread ----
        int v[kApplyItems];
        uint32_t m[kApplyItems], cv[kApplyItems];
        int deg[kApplyItems], rs[kApplyItems];
#pragma unroll
        for (int j = 0; j < kApplyItems; j++) {
          const int idx = b0 + j * kBlock + threadIdx.x;
          v[j] = (idx < cnt) ? s_list[idx] : -1;
          PGX_ASSERT(v[j] < n);
        }
        // every load of the batch in one round trip: the row pointers are
        // read speculatively (the list is in vertex order: near-coalesced)
        int re[kApplyItems];
#pragma unroll
        for (int j = 0; j < kApplyItems; j++) {
          if (v[j] >= 0) {
            m[j] = BFS ? bfs_msg : *slot<S>(mailbox, v[j]);
            cv[j] = *slot<S>(val, v[j]);
            rs[j] = row_ptr[v[j]];
            re[j] = row_ptr[v[j] + 1];
          }
        }
        unsigned long long mine = 0;
#pragma unroll
        for (int j = 0; j < kApplyItems; j++) {
          deg[j] = 0;
          if (v[j] >= 0) {
            if (!BFS) *slot<S>(mailbox, v[j]) = kNeutralMin;  // consume (mailbox.py:112-117)
            if (m[j] < cv[j]) {
              *slot<S>(val, v[j]) = m[j];
              bcast++;
              deg[j] = re[j] - rs[j];
              if (deg[j] > 0) mine += (1ull << 32) | (unsigned long long)deg[j];
            }
          }
        }
        unsigned long long total;
        unsigned long long run = block_excl_scan_u64(mine, s_w, &total);
        if (no_frontier) {
          // CC, next superstep predicted segmented: it reads the send
          // values, not a frontier -- only count (senders << 32 | edges),
          // no frontier SoA / tile map stores
          if (threadIdx.x == 0 && total) atomicAdd(&ctr->packed, total);
#pragma unroll
          for (int j = 0; j < kApplyItems; j++)
            if (deg[j] > 0) sv[v[j]] = m[j];
          continue;
        }
        if (total != 0) {  // block-uniform
          if (threadIdx.x == 0) s_gbase = atomicAdd(&ctr->packed, total);
          __syncthreads();
          run += s_gbase;
#pragma unroll
          for (int j = 0; j < kApplyItems; j++) {
            if (deg[j] > 0) {
              // senders bitmap of the next superstep (segmented scatter)
              if (snd) red_or_b32(snd + (v[j] >> 5), 1u << (v[j] & 31));
              if (sv) sv[v[j]] = m[j];  // CC: the label it sends
              const unsigned pos = (unsigned)(run >> 32);
              const int eb = (int)(run & 0xFFFFFFFFull);
              PGX_ASSERT(pos < (unsigned)n && (int64_t)eb + deg[j] <= (int64_t)INT32_MAX);
              ws.f_eb[pos] = eb;
              ws.f_rs[pos] = rs[j];
              f_msg[pos] = (APP == PGX_APP_SSSP) ? m[j] + 1u : m[j];
              for (int64_t t = ((int64_t)eb + kTile - 1) / kTile; t * kTile < (int64_t)eb + deg[j];
                   t++)
                ws.tile_src[t] = (int)pos;
              run += (1ull << 32) | (unsigned long long)deg[j];
            }
          }
        }
      }
      __syncthreads();  // s_list reuse
    }
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


}  // namespace pgx
