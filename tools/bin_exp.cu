// bin_exp.cu -- EXPERIMENT (not part of libpgx): propagation blocking for
// the dense min scatter.  Phase A stages (dst, msg) pairs in shared memory
// by destination bin and writes each bin's run with coalesced stores into
// a per-bin region (capacity = the bin's total in-degree); phase B
// min-combines a bin chunk in a shared-memory copy of the bin's vertex
// range and flushes it with coalesced red.min + ballot has-words.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -Xcompiler -fPIC -shared -Iinclude tools/bin_exp.cu -o exp/libbinexp.so
#include "../paper_2010_01542_b200/csrc/pgx_common.cuh"

using namespace pgx;

namespace {

#ifndef BINEXP_A_BLOCKS
#define BINEXP_A_BLOCKS 2
#endif
constexpr int kBinShift = 13;
constexpr int kBinV = 1 << kBinShift;
constexpr int kMaxBins = 1024;
constexpr int kBatch = kWarps * kTile;  // 4096 edges per CTA batch

__device__ __forceinline__ unsigned block_excl_scan_u32(unsigned x, unsigned *s_w,
                                                        unsigned *total) {
  unsigned incl = x;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if ((int)lane_id() >= o) incl += y;
  }
  if (lane_id() == 31) s_w[threadIdx.x >> 5] = incl;
  __syncthreads();
  if (threadIdx.x < 32) {
    const unsigned w = (threadIdx.x < kWarps) ? s_w[threadIdx.x] : 0u;
    unsigned wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if ((int)threadIdx.x >= o) wi += y;
    }
    if (threadIdx.x < kWarps) s_w[threadIdx.x] = wi - w;
    if (threadIdx.x == 31) s_w[32] = wi;
  }
  __syncthreads();
  const unsigned r = s_w[threadIdx.x >> 5] + incl - x;
  *total = s_w[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kBlock, BINEXP_A_BLOCKS)
    bin_kernel(const int32_t *col, const int32_t *eb, const int32_t *ids, const int32_t *tile_src,
               int32_t nsrc, int64_t E, int32_t nbins, const int64_t *bin_base, unsigned *cursor,
               uint2 *pairs) {
  extern __shared__ __align__(16) char smem[];
  __shared__ unsigned s_w[33];
  const int lane = (int)lane_id();
  const int warp = threadIdx.x >> 5;
  int32_t *s_eb = reinterpret_cast<int32_t *>(smem) + warp * kSlots;
  uint32_t *s_msg = reinterpret_cast<uint32_t *>(smem + sizeof(int32_t) * kWarps * kSlots) +
                    warp * kSlots;
  unsigned *s_cnt = reinterpret_cast<unsigned *>(smem + 8 * kWarps * kSlots);
  unsigned *s_off = s_cnt + kMaxBins;
  unsigned *s_gpos = s_off + kMaxBins;
  uint2 *s_stage = reinterpret_cast<uint2 *>(s_gpos + kMaxBins);
  const uint64_t pol = evict_first_policy();
  const unsigned upto = (lane == 31) ? 0xFFFFFFFFu : ((2u << lane) - 1u);
  const int64_t ntiles = (E + kTile - 1) / kTile;
  const int64_t nbatch = (ntiles + kWarps - 1) / kWarps;

  for (int64_t bt = blockIdx.x; bt < nbatch; bt += gridDim.x) {
    for (int b = threadIdx.x; b < nbins; b += kBlock) s_cnt[b] = 0u;
    const int64_t t = bt * kWarps + warp;
    int w[kItems];
    uint32_t mv[kItems];
    unsigned pos[kItems];
#pragma unroll
    for (int r = 0; r < kItems; r++) w[r] = -1;
    if (t < ntiles) {
      const int64_t e0 = t * kTile;
      const int64_t e1 = min(E, e0 + kTile);
      const int i0 = tile_src[t];
      const int i1 = (t + 1 < ntiles) ? tile_src[t + 1] : nsrc - 1;
      const int k = i1 - i0 + 1;
      for (int j = lane; j <= k; j += 32) {
        const int i = i0 + j;
        if (j < k) {
          s_eb[j] = eb[i];
          s_msg[j] = (uint32_t)ids[i];
        } else {
          s_eb[j] = (i < nsrc) ? eb[i] : (int32_t)E;
        }
      }
      __syncwarp();
      int cur = 0;
#pragma unroll
      for (int r = 0; r < kItems; r++) {
        const int64_t base = e0 + r * 32;
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
        if (e < e1) {
          mv[r] = s_msg[src];
          w[r] = ld_stream(col + e, pol);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kItems; r++)
      if (w[r] >= 0) pos[r] = atomicAdd(&s_cnt[w[r] >> kBinShift], 1u);
    __syncthreads();
    // exclusive scan of the bin counts (nbins <= 2 per thread)
    const int b0 = 2 * threadIdx.x;
    const unsigned c0 = (b0 < nbins) ? s_cnt[b0] : 0u, c1 = (b0 + 1 < nbins) ? s_cnt[b0 + 1] : 0u;
    unsigned total;
    const unsigned ex = block_excl_scan_u32(c0 + c1, s_w, &total);
    if (b0 < nbins) {
      s_off[b0] = ex;
      if (c0) s_gpos[b0] = atomicAdd(cursor + b0, c0);
    }
    if (b0 + 1 < nbins) {
      s_off[b0 + 1] = ex + c0;
      if (c1) s_gpos[b0 + 1] = atomicAdd(cursor + b0 + 1, c1);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kItems; r++)
      if (w[r] >= 0) s_stage[s_off[w[r] >> kBinShift] + pos[r]] = make_uint2((unsigned)w[r], mv[r]);
    __syncthreads();
    for (unsigned i = threadIdx.x; i < total; i += kBlock) {
      const uint2 p = s_stage[i];
      const int b = (int)(p.x >> kBinShift);
      pairs[bin_base[b] + s_gpos[b] + (i - s_off[b])] = p;
    }
    __syncthreads();
  }
}

// one work item = (bin, first pair, last pair) of that bin's region
__global__ void __launch_bounds__(kBlock, 2)
    combine_kernel(const uint2 *pairs, const int64_t *bin_base, const int4 *items, int32_t nitems,
                   int32_t n, uint32_t *mailbox, uint32_t *has) {
  __shared__ uint32_t s_mb[kBinV];
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int4 item = items[it];
    const int b = item.x;
    const int vlo = b << kBinShift;
    for (int v = threadIdx.x; v < kBinV; v += kBlock) s_mb[v] = kNeutralMin;
    __syncthreads();
    const uint2 *pp = pairs + bin_base[b];
    for (int i = item.y + threadIdx.x; i < item.z; i += kBlock) {
      const uint2 p = pp[i];
      const int o = (int)p.x - vlo;
      if (p.y < s_mb[o]) atomicMin(&s_mb[o], p.y);
    }
    __syncthreads();
    for (int v = threadIdx.x; v < kBinV; v += kBlock) {
      const int vv = vlo + v;
      const uint32_t x = (vv < n) ? s_mb[v] : kNeutralMin;
      if (x != kNeutralMin) red_min_u32(mailbox + vv, x);
      const unsigned bits = __ballot_sync(0xFFFFFFFFu, x != kNeutralMin);
      if (lane_id() == 0 && bits) red_or_b32(has + (vv >> 5), bits);
    }
    __syncthreads();
  }
}

}  // namespace

extern "C" {

int binexp_phase_a(const int32_t *col, const int32_t *eb, const int32_t *ids,
                   const int32_t *tile_src, int32_t nsrc, int64_t E, int32_t nbins,
                   const int64_t *bin_base, unsigned *cursor, void *pairs, int32_t grid,
                   uintptr_t stream) {
  if (nbins > kMaxBins) return -1;
  const size_t smem = 8 * kWarps * kSlots + 3 * 4 * kMaxBins + 8 * kBatch;
  cudaFuncSetAttribute(bin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bin_kernel<<<grid, kBlock, smem, (cudaStream_t)stream>>>(col, eb, ids, tile_src, nsrc, E, nbins,
                                                           bin_base, cursor, (uint2 *)pairs);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

int binexp_phase_b(const void *pairs, const int64_t *bin_base, const void *items, int32_t nitems,
                   int32_t n, uint32_t *mailbox, uint32_t *has, int32_t grid, uintptr_t stream) {
  combine_kernel<<<grid, kBlock, 0, (cudaStream_t)stream>>>(
      (const uint2 *)pairs, bin_base, (const int4 *)items, nitems, n, mailbox, has);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

int binexp_smem_a(size_t *bytes) {
  *bytes = 8 * kWarps * kSlots + 3 * 4 * kMaxBins + 8 * kBatch;
  return 0;
}
}
