// pgx_microbench.cu -- the scattered-access ceilings of this path
// ("secondary ceiling, to be measured by the builder:
// random-address L2 atomic throughput (atomicMin.u32, red.add.f64)").
//
// Every superstep kernel of libpgx is bound by 4-8 byte accesses to
// uniformly random vertex slots (mailbox combines, read-filters, share
// gathers) rather than by streaming HBM bandwidth.  These kernels measure
// the best rate the B200 sustains for each access kind, with addresses from
// a counter hash (no index traffic), 8 independent accesses in flight per
// thread and a persistent grid -- the denominator for the kernels' second
// roofline.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/pgx.h"

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <int KIND>
__global__ void __launch_bounds__(256) random_access_kernel(void *buf, uint64_t mask,
                                                          int64_t ops_per_thread, uint64_t seed,
                                                          unsigned long long *sink) {
  const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t *u = reinterpret_cast<uint32_t *>(buf);
  double *d = reinterpret_cast<double *>(buf);
  unsigned long long acc = 0;
  double dacc = 0.0;
  for (int64_t i = 0; i < ops_per_thread; i += 8) {
    uint64_t idx[8];
#pragma unroll
    for (int j = 0; j < 8; j++) idx[j] = mix64(seed ^ ((gtid << 24) + (uint64_t)(i + j))) & mask;
    if (KIND == PGX_MB_LOAD_U32) {
      uint32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; j++) v[j] = u[idx[j]];
#pragma unroll
      for (int j = 0; j < 8; j++) acc += v[j];
    } else if (KIND == PGX_MB_LOAD_F64) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; j++) v[j] = __ldg(d + idx[j]);
#pragma unroll
      for (int j = 0; j < 8; j++) dacc += v[j];
    } else if (KIND == PGX_MB_LOAD_U32_CG || KIND == PGX_MB_LOAD_U32_NA ||
               KIND == PGX_MB_LOAD_U32_RELAXED) {
      uint32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; j++) {
        if (KIND == PGX_MB_LOAD_U32_CG)
          asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v[j]) : "l"(u + idx[j]));
        else if (KIND == PGX_MB_LOAD_U32_NA)
          asm volatile("ld.global.L1::no_allocate.u32 %0, [%1];" : "=r"(v[j]) : "l"(u + idx[j]));
        else
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v[j]) : "l"(u + idx[j]));
      }
#pragma unroll
      for (int j = 0; j < 8; j++) acc += v[j];
    } else if (KIND == PGX_MB_RED_MIN_U32) {
#pragma unroll
      for (int j = 0; j < 8; j++)
        asm volatile("red.relaxed.gpu.global.min.u32 [%0], %1;" ::"l"(u + idx[j]),
                     "r"((uint32_t)idx[j]) : "memory");
    } else if (KIND == PGX_MB_RED_ADD_F64) {
#pragma unroll
      for (int j = 0; j < 8; j++) atomicAdd(d + idx[j], 1.0);
    } else if (KIND == PGX_MB_ATOM_MIN_U32) {
      uint32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; j++) v[j] = atomicMin(u + idx[j], (uint32_t)idx[j]);
#pragma unroll
      for (int j = 0; j < 8; j++) acc += v[j];
    }
  }
  if (acc + (unsigned long long)dacc == 0x123456789ull) atomicAdd(sink, 1ull);  // keep loads live
}

template <int KIND>
cudaError_t launch(void *buf, uint64_t mask, int64_t per_thread, uint64_t seed,
                   unsigned long long *sink, int grid, cudaStream_t st) {
  random_access_kernel<KIND><<<grid, 256, 0, st>>>(buf, mask, per_thread, seed, sink);
  return cudaGetLastError();
}

}  // namespace

extern "C" int pgx_microbench(int kind, void *buf, int64_t n_elems, int64_t n_ops,
                              uint64_t seed, float *ms, uintptr_t stream) {
  if (!buf || !ms || n_elems < 2 || (n_elems & (n_elems - 1)) || n_ops < 1) return PGX_EINVAL;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return PGX_ECUDA;
  const int grid = sms * 8;
  const int64_t threads = (int64_t)grid * 256;
  int64_t per_thread = (n_ops + threads - 1) / threads;
  per_thread = (per_thread + 7) / 8 * 8;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long *sink = nullptr;
  if (cudaMalloc(&sink, sizeof(unsigned long long)) != cudaSuccess) return PGX_ECUDA;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const uint64_t mask = (uint64_t)n_elems - 1;
  cudaError_t e = cudaSuccess;
  for (int rep = 0; rep < 2 && e == cudaSuccess; rep++) {  // warm-up + timed
    cudaEventRecord(a, st);
    switch (kind) {
      case PGX_MB_LOAD_U32: e = launch<PGX_MB_LOAD_U32>(buf, mask, per_thread, seed, sink, grid, st); break;
      case PGX_MB_LOAD_F64: e = launch<PGX_MB_LOAD_F64>(buf, mask, per_thread, seed, sink, grid, st); break;
      case PGX_MB_RED_MIN_U32: e = launch<PGX_MB_RED_MIN_U32>(buf, mask, per_thread, seed, sink, grid, st); break;
      case PGX_MB_RED_ADD_F64: e = launch<PGX_MB_RED_ADD_F64>(buf, mask, per_thread, seed, sink, grid, st); break;
      case PGX_MB_ATOM_MIN_U32: e = launch<PGX_MB_ATOM_MIN_U32>(buf, mask, per_thread, seed, sink, grid, st); break;
      case PGX_MB_LOAD_U32_CG: e = launch<PGX_MB_LOAD_U32_CG>(buf, mask, per_thread, seed, sink, grid, st); break;
      case PGX_MB_LOAD_U32_NA: e = launch<PGX_MB_LOAD_U32_NA>(buf, mask, per_thread, seed, sink, grid, st); break;
      case PGX_MB_LOAD_U32_RELAXED: e = launch<PGX_MB_LOAD_U32_RELAXED>(buf, mask, per_thread, seed, sink, grid, st); break;
      default: e = cudaErrorInvalidValue;
    }
    cudaEventRecord(b, st);
  }
  if (e == cudaSuccess) e = cudaEventSynchronize(b);
  if (e == cudaSuccess) e = cudaEventElapsedTime(ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  return e == cudaSuccess ? PGX_OK : PGX_ECUDA;
}
