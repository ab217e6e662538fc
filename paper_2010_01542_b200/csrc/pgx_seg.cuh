// pgx_seg.cuh -- K1s, the destination-segmented scatter for dense supersteps:
// every recipient combines in shared memory.  Reference: the same
// send_to_out_neighbors / send_hybrid path as K1 (engine.py:154-162,
// mailbox.py:180-199), with the paper's hybrid combiner taken to its end:
// instead of pre-combining only hub recipients in shared memory
// (mailbox.py:180-199's lock-free / locked split), a dense superstep
// combines EVERY message in a shared-memory copy of its recipient's
// mailbox segment, and only the combined slot leaves the SM.
//
// Why (profiles/ceilings_r2_sweep.jsonl): a random 4-byte
// access that misses L1 costs one L1->L2 request, and an SM issues at most
// one per clock (290 G/s on B200 whatever the occupancy or loads in
// flight).  K1 pays >= 1 such request per edge (its read-filter).  Here the
// edges are regrouped by destination segment (S = 2^seg_log2 consecutive
// vertex ids; pgx_seg_build): inside a segment they stay in CSR order, so
// an entry (source, first edge) covers a source's whole run of edges into
// the segment and each destination is a 16-bit offset.  The per-edge work
// becomes a streamed 2-byte load plus a shared-memory filter / atomicMin;
// the random global accesses drop to one message lookup per entry
// (C2 2.3, C5 1.8 edges per entry at S = 8192) and none in CC superstep 0,
// whose messages are the source ids.
//
// Work: items (a segment, or a slice of a hot one: R-MAT puts a large share
// of the edges into the low-id segments) are claimed from a per-superstep
// counter, largest first.  A CTA clears its smem segment, its warps walk
// the item's 256-edge tiles (one cp.async round trip per tile for the
// destinations and the entry window; sources found with the REDUX boundary
// trick of K1), then the CTA flushes: an item that owns its segment stores
// the slots and the has-bitmask words (one per warp) directly; slices of a
// hot segment combine with coalesced fire-and-forget red.min and one
// warp-aggregated red.or per has word.  The result is exactly K1's
// mailbox + has-bitmask, so K2 (apply) runs unchanged.
#pragma once

#include <type_traits>

#include "pgx_common.cuh"

namespace pgx {

__device__ __forceinline__ void cp_async4(void *sdst, const void *gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(void *sdst, const void *gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// Messages of a segmented scatter pass:
//   kSegSourceId  CC superstep 0: every source sends its id;
//   kSegLabel     the source sends sv[src], its send value of this
//                 superstep (the neutral when it is not a sender: a no-op);
//   kSegUniform   the sources flagged in the senders bitmap send `uniform`
//                 (the first unit-weight SSSP form, kept for A/B builds: the
//                 run kernel now feeds SSSP send values to kSegLabel).
enum SegMsg { kSegSourceId = 0, kSegLabel = 1, kSegUniform = 2 };

// work items: about kSegItemsPerCta per persistent CTA, and never more than
// kMaxSegSlices slices of hot segments in total (pgx_seg_build)
constexpr int kSegItemsPerCta = 2;
constexpr int64_t kMaxSegSlices = 4096;
// col16: bit 15 flags the first edge of an entry, the low seg_log2 bits
// are the destination's offset in its segment (so seg_log2 <= 15)
constexpr uint32_t kSegEntryFlag = 0x8000u;
constexpr int kSegMaxLog2 = 15;

struct SegPass {
  PgxSegIndex ix;
  int64_t m;
  int32_t n;
  const uint32_t *snd;  // kSegUniform: senders bitmap of this superstep
  const uint32_t *sv;   // kSegLabel: send values of this superstep
  uint32_t uniform;     // kSegUniform: the message
  uint32_t *mailbox;    // K1's outputs: min-combined mailbox + has-bitmask
  uint32_t *has;
  unsigned *item_ctr;   // zero before the pass
  bool write_mailbox;   // false: the has-bitmask is the whole result (unit SSSP)
  int32_t id_offset;    // kSegSourceId: message = entry source + id_offset
  uint32_t out_neutral; // what an owned, untouched slot is stored as (the
                        // partitioned path's exchange neutral, INT32_MAX)
};

// Shared-memory slot of segment offset `loc`: the bank bits (low 5) are
// XORed with a hash of the rest.  R-MAT offsets are skewed towards zero
// bits (P(bit = 0) = a + c = 0.76), so a quarter of a round's lanes would
// share bank 0 -- 7.5-way conflicts measured on C5 (ncu, superstep 0).  A
// bijection within each 32-slot row: a warp's flush of 32 consecutive
// slots still reads one row, conflict-free.
__device__ __forceinline__ int seg_swz(int loc) {
  return loc ^ (int)(((uint32_t)(loc >> 5) * 0x9E3779B1u) >> 27);
}

// per-warp window: the messages of the tile's entries [kSegMsgSlots], the
// tile's flagged 16-bit destinations [kTile]; 16-byte aligned (cp.async 16)
constexpr int kSegMsgSlots = (kSlots + 3) & ~3;
constexpr int kSegWinWords = kSegMsgSlots + kTile / 2;
static_assert(kSegWinWords % 4 == 0, "16-byte aligned per-warp windows");

__host__ __device__ constexpr size_t seg_smem_bytes(int seg_log2) {
  return ((size_t)4 << seg_log2) + (size_t)kWarps * kSegWinWords * 4;
}

// superstep 0 of CC (messages = source ids, no send-value loads) is bound
// by instruction issue: two edges per lane and round there (C5 superstep 0
// 2.75 -> 2.71 ms, the run -0.6 %); the label supersteps keep one edge per
// lane (pairs measured 5 % slower there: 4.12 vs 3.92 ms on C5), four per
// lane for superstep 0 measured the same as two
#ifndef PGX_SEG_PAIRS
#define PGX_SEG_PAIRS 1
#endif

template <int MSG>
__device__ void seg_scatter_phase(const SegPass &a, char *smem_raw) {
  uint32_t *smem = reinterpret_cast<uint32_t *>(smem_raw);
  const int L = a.ix.seg_log2;
  const int S = 1 << L;
  const uint32_t lmask = (uint32_t)S - 1u;
  uint32_t *s_mb = smem;  // [S] this item's mailbox segment
  __shared__ int s_item[4];
  __shared__ unsigned s_tctr;
  const int lane = (int)lane_id(), warp = threadIdx.x >> 5;
  uint32_t *w_msg = smem + S + warp * kSegWinWords;
  uint16_t *w_col = reinterpret_cast<uint16_t *>(w_msg + kSegMsgSlots);
  const unsigned upto = (lane == 31) ? 0xFFFFFFFFu : ((2u << lane) - 1u);
  const int ntiles = (int)((a.m + kTile - 1) / kTile);
  const int nent = a.ix.nent;
  for (;;) {
    if (threadIdx.x == 0) {
      const int it = (int)atomicAdd(a.item_ctr, 1u);
      s_item[0] = it;
      if (it < a.ix.nitems) {
        const int4 d = reinterpret_cast<const int4 *>(a.ix.items)[it];
        s_item[1] = d.x;
        s_item[2] = d.y;
        s_item[3] = d.z;
        s_tctr = (unsigned)d.w << 31;  // bit 31: the item owns its segment
      }
    }
    for (int i = threadIdx.x; i < S; i += blockDim.x) s_mb[i] = kNeutralMin;
    __syncthreads();
    if (s_item[0] >= a.ix.nitems) break;  // block-uniform
    const int seg = s_item[1], e0 = s_item[2], e1 = s_item[3];
    const bool sole = (s_tctr >> 31) != 0u;
    __syncthreads();
    if (threadIdx.x == 0) s_tctr = 0u;
    __syncthreads();
    const int t0 = e0 / kTile, t1 = (e1 + kTile - 1) / kTile;
    auto claim = [&]() -> int {
      unsigned c = 0;
      if (lane == 0) c = atomicAdd(&s_tctr, 1u);
      c = __shfl_sync(0xFFFFFFFFu, c, 0);
      return t0 + (int)c < t1 ? t0 + (int)c : -1;
    };
    int t = claim();
    int i0n = 0, i1n = 0;
    if (t >= 0) {
      i0n = a.ix.tile_ent[t];
      i1n = (t + 1 < ntiles) ? a.ix.tile_ent[t + 1] : nent - 1;
    }
    while (t >= 0) {
      const int i0 = i0n, i1 = i1n;
      const int tn = claim();
      if (tn >= 0) {  // the next tile's entry range is in flight during this one
        i0n = a.ix.tile_ent[tn];
        i1n = (tn + 1 < ntiles) ? a.ix.tile_ent[tn + 1] : nent - 1;
      }
      const int ta = t * kTile;
      const int ea = max(e0, ta) - ta, ez = min(e1, ta + kTile) - ta;  // tile-relative
      const int k = i1 - i0 + 1;  // <= kTile + 1 entries
      PGX_ASSERT(i0 >= 0 && k >= 1 && k <= kTile + 1 && i1 < nent);
      __syncwarp();
      // one round trip for the whole tile: the flagged 16-bit destinations
      // and the entries' messages
      cp_async16(w_col + lane * 8, a.ix.col16 + ta + lane * 8);
      if (MSG == kSegSourceId && a.id_offset == 0) {
#pragma unroll
        for (int q = 0; q < (kSlots + 31) / 32; q++) {
          const int j = lane + 32 * q;
          if (j < k) cp_async4(w_msg + j, a.ix.ent_src + i0 + j);
        }
      } else if (MSG == kSegSourceId) {  // a rank's slice: global source ids
#pragma unroll
        for (int q = 0; q < (kSlots + 31) / 32; q++) {
          const int j = lane + 32 * q;
          if (j < k) w_msg[j] = (uint32_t)(__ldg(a.ix.ent_src + i0 + j) + a.id_offset);
        }
      } else {
        int src[(kSlots + 31) / 32];
#pragma unroll
        for (int q = 0; q < (kSlots + 31) / 32; q++) {
          const int j = lane + 32 * q;
          src[q] = (j < k) ? __ldg(a.ix.ent_src + i0 + j) : -1;
        }
        if (MSG == kSegLabel) {
          // one random load per entry: the send value is the neutral for
          // a source that does not send in this superstep
#pragma unroll
          for (int q = 0; q < (kSlots + 31) / 32; q++)
            if (src[q] >= 0) cp_async4(w_msg + lane + 32 * q, a.sv + src[q]);
        } else {
          uint32_t bits[(kSlots + 31) / 32];
#pragma unroll
          for (int q = 0; q < (kSlots + 31) / 32; q++)
            bits[q] = src[q] >= 0 ? a.snd[src[q] >> 5] : 0u;
#pragma unroll
          for (int q = 0; q < (kSlots + 31) / 32; q++) {
            const int j = lane + 32 * q;
            if (j < k) w_msg[j] = ((bits[q] >> (src[q] & 31)) & 1u) ? a.uniform : kNeutralMin;
          }
        }
      }
      cp_async_wait_all();
      __syncwarp();
      // entry of edge e (tile-relative) = flags in [0, e] - flag(0): the
      // tile's first edge belongs to entry i0 whether or not it starts it
      int cur = -(int)(w_col[0] >> 15);
      // the destinations are stored pre-swizzled (seg_swz, pgx_seg_build)
      auto rounds = [&](auto checked) {
#pragma unroll
        for (int r = 0; r < kItems; r++) {
          const int el = r * 32 + lane;
          const uint32_t c = w_col[el];
          const unsigned bm = __ballot_sync(0xFFFFFFFFu, (c & kSegEntryFlag) != 0u);
          const int sidx = cur + __popc(bm & upto);
          cur += __popc(bm);
          if (!decltype(checked)::value || (el >= ea && el < ez)) {
            PGX_ASSERT(sidx >= 0 && sidx < k);
            const uint32_t msg = w_msg[sidx];
            const int loc = (int)(c & lmask);
            // shared-memory read-filter (the mailbox.py:159 short-circuit),
            // then the combine; both on the SM, no L2 request
            if (msg < s_mb[loc]) atomicMin(s_mb + loc, msg);
          }
        }
      };
#if PGX_SEG_PAIRS
      // two consecutive edges per lane and round (one 32-bit destination
      // pair load, one ballot per edge parity): 64 edges per round, for the
      // source-id superstep
      const uint32_t lt = (1u << lane) - 1u;  // lanes below this one
      auto rounds2 = [&](auto checked) {
        const uint32_t *w_col2 = reinterpret_cast<const uint32_t *>(w_col);
#pragma unroll
        for (int r = 0; r < kItems / 2; r++) {
          const int el = r * 64 + 2 * lane;
          const uint32_t cc = w_col2[r * 32 + lane];
          const uint32_t c0 = cc & 0xFFFFu, c1 = cc >> 16;
          const bool f0 = (c0 & kSegEntryFlag) != 0u, f1 = (c1 & kSegEntryFlag) != 0u;
          const unsigned b0 = __ballot_sync(0xFFFFFFFFu, f0);
          const unsigned b1 = __ballot_sync(0xFFFFFFFFu, f1);
          const int sidx0 = cur + __popc(b0 & (lt | (1u << lane))) + __popc(b1 & lt);
          const int sidx1 = sidx0 + (int)f1;
          cur += __popc(b0) + __popc(b1);
          if (!decltype(checked)::value || (el >= ea && el < ez)) {
            const uint32_t msg = w_msg[sidx0];
            const int loc = (int)(c0 & lmask);
            if (msg < s_mb[loc]) atomicMin(s_mb + loc, msg);
          }
          if (!decltype(checked)::value || (el + 1 >= ea && el + 1 < ez)) {
            const uint32_t msg = w_msg[sidx1];
            const int loc = (int)(c1 & lmask);
            if (msg < s_mb[loc]) atomicMin(s_mb + loc, msg);
          }
        }
      };
      if (MSG != kSegSourceId) {
        if (ea == 0 && ez == kTile) rounds(std::false_type{});  // interior tile
        else rounds(std::true_type{});
      } else if (ea == 0 && ez == kTile) {
        rounds2(std::false_type{});
      } else {
        rounds2(std::true_type{});
      }
#else
      if (ea == 0 && ez == kTile) rounds(std::false_type{});  // interior tile
      else rounds(std::true_type{});
#endif
      t = tn;
    }
    __syncthreads();
    // flush: 32 consecutive slots per warp = one has-bitmask word
    const int base = seg << L;
#pragma unroll 4
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
      const uint32_t v = s_mb[seg_swz(i)];
      const int g = base + i;
      const bool in = g < a.n;
      const bool touched = v != kNeutralMin && in;
      const unsigned bits = __ballot_sync(0xFFFFFFFFu, touched);
      if (sole) {  // the item owns these slots and words: plain stores
        if (a.write_mailbox && in) a.mailbox[g] = touched ? v : a.out_neutral;
        if (lane == 0 && in) a.has[g >> 5] = bits;
      } else {     // a slice of a hot segment: fire-and-forget combines
        if (a.write_mailbox && touched) red_min_u32(a.mailbox + g, v);
        if (lane == 0 && bits) red_or_b32(a.has + (g >> 5), bits);
      }
    }
    __syncthreads();
  }
}

}  // namespace pgx
