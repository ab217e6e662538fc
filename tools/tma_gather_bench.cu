// tma_gather_bench.cu -- can the TMA unit add random-gather throughput on
// top of the LSU path? (experiment, not part of libpgx)
//
// The pull fold and the segmented scatter are bound by scattered 8-byte
// loads: one L1TEX tag lookup per distinct line, ~1 per SM clock (DESIGN.md
// 3).  A bulk copy (cp.async.bulk, the TMA engine) fetches global memory
// into shared memory without the LSU / L1 tag stage.  This measures random
// 16-byte gathers per second over the whole GPU for
//   mode 0: LSU only    (ld.global.nc.v2.f64, F in flight per thread)
//   mode 1: TMA only    (cp.async.bulk 16 B per gather into shared memory,
//                        one mbarrier per warp)
//   mode 2: both        (half of each lane's gathers on each path)
// over an L2-resident (32 MB) and an HBM-resident (1 GB) array.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ab/tma_gather_bench tools/tma_gather_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int kThreads = 1024;
constexpr int kF = 8;  // gathers per lane and iteration

__device__ __forceinline__ uint32_t hash32(uint32_t a, uint32_t b) {
  uint32_t h = a * 0x9E3779B1u ^ b * 0x85EBCA77u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  h *= 0x297A2D39u;
  h ^= h >> 15;
  return h;
}

__device__ __forceinline__ void mbar_init(uint64_t *m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(m)),
               "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t *m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(m)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W;\n"
      "}\n" ::"r"((unsigned)__cvta_generic_to_shared(m)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk16(void *dst, const void *src, uint64_t *m) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(src), "r"((unsigned)__cvta_generic_to_shared(m))
      : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) gather_kernel(const double2 *buf, uint32_t mask,
                                                             int iters, double *sink) {
  extern __shared__ __align__(16) char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem) + warp;
  double2 *land = reinterpret_cast<double2 *>(smem + 32 * 8) + warp * 32 * kF;
  if (lane == 0) mbar_init(mbar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const uint32_t tid = blockIdx.x * kThreads + threadIdx.x;
  constexpr int kT = MODE == 0 ? 0 : MODE == 1 ? kF : kF / 2;  // gathers on the TMA path
  double acc = 0.0;
  unsigned phase = 0;
  for (int it = 0; it < iters; it++) {
    if (kT > 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_expect(mbar, 32u * kT * 16u);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < kT; j++) {
        const uint32_t i = hash32(tid, (uint32_t)(it * kF + j)) & mask;
        bulk16(land + lane * kF + j, buf + i, mbar);
      }
    }
    double2 v[kF - kT > 0 ? kF - kT : 1];
#pragma unroll
    for (int j = 0; j < kF - kT; j++) {
      const uint32_t i = hash32(tid, (uint32_t)(it * kF + kT + j)) & mask;
      v[j] = __ldg(buf + i);
    }
#pragma unroll
    for (int j = 0; j < kF - kT; j++) acc += v[j].x;
    if (kT > 0) {
      mbar_wait(mbar, phase);
      phase ^= 1u;
#pragma unroll
      for (int j = 0; j < kT; j++) acc += land[lane * kF + j].x;
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 32 * 8 + (size_t)32 * 32 * kF * 16;  // 131 KB
  double *sink;
  cudaMalloc(&sink, 8);
  for (size_t bytes : {(size_t)32 << 20, (size_t)1 << 30}) {
    double2 *buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    const uint32_t mask = (uint32_t)(bytes / 16 - 1);
    for (int mode = 0; mode < 3; mode++) {
      void (*k)(const double2 *, uint32_t, int, double *) =
          mode == 0 ? gather_kernel<0> : mode == 1 ? gather_kernel<1> : gather_kernel<2>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int iters = 200;
      k<<<sms, kThreads, smem>>>(buf, mask, 10, sink);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      k<<<sms, kThreads, smem>>>(buf, mask, iters, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const cudaError_t e = cudaGetLastError();
      const double g = (double)sms * kThreads * iters * kF / (ms * 1e-3) / 1e9;
      printf("{\"array_mb\": %zu, \"mode\": \"%s\", \"ms\": %.3f, \"G_gathers_per_s\": %.1f, "
             "\"per_sm_clk_at_1965MHz\": %.3f, \"err\": \"%s\"}\n",
             bytes >> 20, mode == 0 ? "lsu" : mode == 1 ? "tma" : "lsu+tma", ms, g,
             g / (sms * 1.965), cudaGetErrorString(e));
    }
    cudaFree(buf);
  }
  return 0;
}
