// seg_exp.cu -- experiment: destination-segmented dense scatter (CC superstep
// 0) with a shared-memory combiner, against the shipped global-filter scatter.
//
// The edges are regrouped by destination segment (S consecutive vertex ids);
// inside a segment they stay in (source, destination) order, so one entry
// (source, first edge) covers all of a source's edges into the segment and
// the destinations are 16-bit offsets.  A CTA takes a work item (a segment,
// or a slice of a hot segment), combines its messages in a shared-memory
// copy of the segment's mailbox (read-filter + atomicMin on smem), then
// flushes the touched slots to the global mailbox with coalesced red.min
// and one ballot-aggregated red.or per has-bitmask word.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared \
//      -o exp/libseg.so tools/seg_exp.cu
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
constexpr int kBlock = 512;
constexpr int kWarps = kBlock / 32;
constexpr int kTile = 256;
constexpr int kSlots = kTile + 2;
constexpr uint32_t kNeutral = 0xFFFFFFFFu;

__device__ __forceinline__ void red_min_u32(uint32_t *p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.min.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_or_b32(uint32_t *p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned short ld_stream_u16(const unsigned short *p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}

struct SegArgs {
  const int32_t *ent_src;   // [nent] source of each entry
  const int32_t *ent_eb;    // [nent + 1] first edge of each entry (segment-grouped edge order)
  const uint16_t *col16;    // [m] destination offset inside the segment
  const int32_t *tile_ent;  // [ntiles + 1] entry holding edge t * kTile
  const int32_t *items;     // [nitems][4] (segment, e0, e1, sole)
  int32_t nitems;
  int32_t nent;
  int64_t m;
  int32_t n;
  int32_t seg_log2;
  uint32_t *mailbox;
  uint32_t *has;
  unsigned *item_ctr;
};

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

// per-warp window: entry edge starts [kSlots], entry messages [kSlots],
// the tile's 16-bit destinations [kTile]
constexpr int kWinWords = 2 * kSlots + kTile / 2;

template <int PASS>
__global__ void __launch_bounds__(kBlock, 2) seg_scatter_kernel(SegArgs a) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int S = 1 << a.seg_log2;
  uint32_t *s_mb = smem;  // [S]
  __shared__ int s_item[4];
  __shared__ unsigned s_tctr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t *w_eb = reinterpret_cast<int32_t *>(smem + S) + warp * kWinWords;
  uint32_t *w_msg = reinterpret_cast<uint32_t *>(w_eb + kSlots);
  uint16_t *w_col = reinterpret_cast<uint16_t *>(w_msg + kSlots);
  const unsigned upto = (lane == 31) ? 0xFFFFFFFFu : ((2u << lane) - 1u);
  const int ntiles = (int)((a.m + kTile - 1) / kTile);
  const int m32 = (int)a.m;
  for (;;) {
    if (threadIdx.x == 0) {
      const int it = (int)atomicAdd(a.item_ctr, 1u);
      s_item[0] = it;
      if (it < a.nitems) {
        s_item[1] = a.items[4 * it];
        s_item[2] = a.items[4 * it + 1];
        s_item[3] = a.items[4 * it + 2];
        s_tctr = (unsigned)a.items[4 * it + 3];  // sole flag in bit 31 stored separately below
      }
    }
    for (int i = threadIdx.x; i < S; i += kBlock) s_mb[i] = kNeutral;
    __syncthreads();
    if (s_item[0] >= a.nitems) break;
    const int seg = s_item[1], e0 = s_item[2], e1 = s_item[3];
    const bool sole = s_tctr != 0u;
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
      i0n = a.tile_ent[t];
      i1n = (t + 1 < ntiles) ? a.tile_ent[t + 1] : a.nent - 1;
    }
    while (t >= 0) {
      const int i0 = i0n, i1 = i1n;
      const int tn = claim();
      if (tn >= 0) {  // next tile's entry range: in flight during this tile
        i0n = a.tile_ent[tn];
        i1n = (tn + 1 < ntiles) ? a.tile_ent[tn + 1] : a.nent - 1;
      }
      const int ta = t * kTile;
      const int ea = max(e0, ta) - ta, ez = min(e1, ta + kTile) - ta;  // tile-relative
      const int k = i1 - i0 + 1;
      __syncwarp();
      // one round trip for the whole tile: 16-bit destinations + entries
      cp_async16(w_col + lane * 8, a.col16 + ta + lane * 8);
#pragma unroll
      for (int q = 0; q < (kSlots + 31) / 32; q++) {
        const int j = lane + 32 * q;
        if (j < k) {
          cp_async4(w_eb + j, a.ent_eb + i0 + j);
          cp_async4(w_msg + j, a.ent_src + i0 + j);
        } else if (j == k) {
          if (i0 + j < a.nent) cp_async4(w_eb + j, a.ent_eb + i0 + j);
          else w_eb[j] = m32;
        }
      }
      cp_async_wait_all();
      __syncwarp();
      int cur = 0;
#pragma unroll 1
      for (int pass = 0; pass < 8 / PASS; pass++) {
        int loc[PASS];
        uint32_t msg[PASS];
#pragma unroll
        for (int r = 0; r < PASS; r++) {
          const int rb = (pass * PASS + r) * 32;  // tile-relative round base
          const int el = rb + lane;
          const int ci = cur + 1 + lane;
          unsigned bit = 0;
          if (ci <= k) {
            const unsigned pp = (unsigned)(w_eb[ci] - ta - rb);
            if (pp < 32u) bit = 1u << pp;
          }
          const unsigned bm = __reduce_or_sync(0xFFFFFFFFu, bit);
          const int src = cur + __popc(bm & upto);
          cur += __popc(bm);
          loc[r] = -1;
          if (el >= ea && el < ez) {
            msg[r] = w_msg[src];
            loc[r] = w_col[el];
          }
        }
        uint32_t old[PASS];
#pragma unroll
        for (int r = 0; r < PASS; r++) old[r] = loc[r] >= 0 ? s_mb[loc[r]] : 0u;
#pragma unroll
        for (int r = 0; r < PASS; r++)
          if (loc[r] >= 0 && msg[r] < old[r]) atomicMin(s_mb + loc[r], msg[r]);
      }
      t = tn;
    }
    __syncthreads();
    // flush: 32 consecutive slots per warp = one has-bitmask word.  A segment
    // combined by this item alone owns its slots and words: plain stores.
    // Slices of a hot segment combine with fire-and-forget reds (the
    // has-bit means "received a message": an OR of the slices' touches).
    const int base = seg << a.seg_log2;
#pragma unroll 4
    for (int i = threadIdx.x; i < S; i += kBlock) {
      const uint32_t v = s_mb[i];
      const int g = base + i;
      const bool in = g < a.n;
      const bool touched = v != kNeutral && in;
      const unsigned bits = __ballot_sync(0xFFFFFFFFu, touched);
      if (sole) {
        if (in) a.mailbox[g] = v;
        if (lane == 0 && in) a.has[g >> 5] = bits;
      } else {
        if (touched) red_min_u32(a.mailbox + g, v);
        if (lane == 0 && bits) red_or_b32(a.has + (g >> 5), bits);
      }
    }
    __syncthreads();
  }
}
}  // namespace

extern "C" int seg_scatter(const int32_t *ent_src, const int32_t *ent_eb, const uint16_t *col16,
                           const int32_t *tile_ent, const int32_t *items, int nitems, int nent,
                           int64_t m, int n, int seg_log2, uint32_t *mailbox, uint32_t *has,
                           unsigned *item_ctr, int ctas_per_sm, int pass, uintptr_t stream) {
  SegArgs a{ent_src, ent_eb, col16, tile_ent, items, nitems, nent, m, n, seg_log2,
            mailbox, has, item_ctr};
  const size_t smem = ((size_t)1 << seg_log2) * 4 + (size_t)kWarps * kWinWords * 4;
  void (*kern)(SegArgs) = pass == 4 ? seg_scatter_kernel<4> : pass == 2 ? seg_scatter_kernel<2>
                                                                         : seg_scatter_kernel<8>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  kern<<<sms * ctas_per_sm, kBlock, smem, (cudaStream_t)stream>>>(a);
  return (int)cudaGetLastError();
}
