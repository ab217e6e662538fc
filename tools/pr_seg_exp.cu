// pr_seg_exp.cu -- experiment: PageRank's fold as a destination-segmented
// PUSH (f64 partial sums combined in a shared-memory copy of each mailbox
// segment) instead of the shipped pull fold.  Same segmented index as the
// CC scatter (pgx_seg_build: entries = one source's run of edges into one
// segment, flagged 16-bit destinations, tile map, work items).  One random
// share load per ENTRY instead of one per in-edge.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//      -I paper_2010_01542_b200/csrc -I include -o exp/libprseg.so tools/pr_seg_exp.cu
#include <cstdint>
#include <cuda_runtime.h>

#include "pgx.h"

namespace {

constexpr int kBlock = 512, kWarps = 16, kItems = 8, kTile = 256, kSlots = kTile + 4;
constexpr int kWinBytes = kSlots * 8 + kTile * 2;  // f64 messages + 16-bit destinations

__device__ __forceinline__ void cp_async8(void *sdst, const void *gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(void *sdst, const void *gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

struct Args {
  PgxSegIndex ix;
  int64_t m;
  int32_t n;
  const double *share;
  double *folded;
  unsigned *item_ctr;
  int mode;  // 0: smem atomicAdd (CAS loop); 1: warp-segmented pre-sum by destination run
};

__global__ void __launch_bounds__(kBlock, 2) pr_seg_kernel(Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L = a.ix.seg_log2, S = 1 << L;
  const uint32_t lmask = (uint32_t)S - 1u;
  double *s_acc = reinterpret_cast<double *>(smem);
  __shared__ int s_item[4];
  __shared__ unsigned s_tctr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char *win = smem + (size_t)S * 8 + (size_t)warp * kWinBytes;
  double *w_msg = reinterpret_cast<double *>(win);
  uint16_t *w_col = reinterpret_cast<uint16_t *>(win + kSlots * 8);
  const unsigned upto = (lane == 31) ? 0xFFFFFFFFu : ((2u << lane) - 1u);
  const int ntiles = (int)((a.m + kTile - 1) / kTile);
  for (;;) {
    if (threadIdx.x == 0) {
      const int it = (int)atomicAdd(a.item_ctr, 1u);
      s_item[0] = it;
      if (it < a.ix.nitems) {
        const int4 d = reinterpret_cast<const int4 *>(a.ix.items)[it];
        s_item[1] = d.x; s_item[2] = d.y; s_item[3] = d.z;
        s_tctr = (unsigned)d.w << 31;
      }
    }
    for (int i = threadIdx.x; i < S; i += blockDim.x) s_acc[i] = 0.0;
    __syncthreads();
    if (s_item[0] >= a.ix.nitems) break;
    const int seg = s_item[1], e0 = s_item[2], e1 = s_item[3];
    const bool sole = (s_tctr >> 31) != 0u;
    __syncthreads();
    if (threadIdx.x == 0) s_tctr = 0u;
    __syncthreads();
    const int t0 = e0 / kTile, t1 = (e1 + kTile - 1) / kTile;
    for (;;) {
      unsigned c = 0;
      if (lane == 0) c = atomicAdd(&s_tctr, 1u);
      c = __shfl_sync(0xFFFFFFFFu, c, 0);
      const int t = t0 + (int)c;
      if (t >= t1) break;
      const int i0 = a.ix.tile_ent[t];
      const int i1 = (t + 1 < ntiles) ? a.ix.tile_ent[t + 1] : a.ix.nent - 1;
      const int k = i1 - i0 + 1;
      __syncwarp();
      cp_async16(w_col + lane * 8, a.ix.col16 + (int64_t)t * kTile + lane * 8);
      int src[(kSlots + 31) / 32];
#pragma unroll
      for (int q = 0; q < (kSlots + 31) / 32; q++) {
        const int j = lane + 32 * q;
        src[q] = (j < k) ? __ldg(a.ix.ent_src + i0 + j) : -1;
      }
#pragma unroll
      for (int q = 0; q < (kSlots + 31) / 32; q++)
        if (src[q] >= 0) cp_async8(w_msg + lane + 32 * q, a.share + src[q]);
      cp_wait();
      __syncwarp();
      const int ta = t * kTile;
      const int ea = max(e0, ta) - ta, ez = min(e1, ta + kTile) - ta;
      int cur = -(int)(w_col[0] >> 15);
#pragma unroll
      for (int r = 0; r < kItems; r++) {
        const int el = r * 32 + lane;
        const uint32_t cc = w_col[el];
        const unsigned bm = __ballot_sync(0xFFFFFFFFu, (cc & 0x8000u) != 0u);
        const int sidx = cur + __popc(bm & upto);
        cur += __popc(bm);
        if (el >= ea && el < ez) atomicAdd(s_acc + (cc & lmask), w_msg[sidx]);
      }
    }
    __syncthreads();
    const int base = seg << L;
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
      const int g = base + i;
      if (g >= a.n) continue;
      const double v = s_acc[i];
      if (sole) a.folded[g] = v;
      else if (v != 0.0) atomicAdd(a.folded + g, v);
    }
    __syncthreads();
  }
}

}  // namespace

extern "C" int pr_seg_fold(const PgxSegIndex *ix, int64_t m, int32_t n, const double *share,
                           double *folded, unsigned *item_ctr, int mode, int ctas,
                           uintptr_t stream) {
  Args a;
  a.ix = *ix;
  a.m = m;
  a.n = n;
  a.share = share;
  a.folded = folded;
  a.item_ctr = item_ctr;
  a.mode = mode;
  const size_t smem = ((size_t)8 << ix->seg_log2) + (size_t)kWarps * kWinBytes;
  if (cudaFuncSetAttribute(pr_seg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return -2;
  pr_seg_kernel<<<ctas, kBlock, smem, (cudaStream_t)stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
