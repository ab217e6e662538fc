// ceiling_sweep.cu -- what bounds a random 4-byte access on B200 (experiment,
// not part of libpgx).  Sweeps, for uniformly random slots:
//   * loads in flight per thread (1..16) and resident threads per SM
//     (occupancy), to show whether the ~290 G/s plateau of round 1 is a
//     latency artefact or a throughput limit;
//   * array size (L1-resident 64 KB, L2-resident 16 MB, HBM 1 GB);
//   * lanes per 128-byte line (1 = every lane its own line .. 32 = one line
//     per warp instruction): the rate in distinct lines per second is the
//     L1TEX wavefront limit if it stays flat;
//   * the same accesses to shared memory (ld.shared, atom.shared.min with
//     and without a read filter), the alternative path for a combiner.
// Output: one JSON object per line on stdout.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exp/ceiling_sweep tools/ceiling_sweep.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

enum Kind { kGlobalLoad = 0, kGlobalRedMin = 1, kSmemLoad = 2, kSmemAtomMin = 3, kSmemFilterMin = 4 };

// index of access j of thread t: lanes are grouped `lpl` per 128-byte line
// (32 u32 slots); a group shares one random line, lanes take distinct slots
__device__ __forceinline__ uint32_t slot_of(uint64_t seed, uint64_t t, uint64_t j, uint32_t mask,
                                            int lpl) {
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t grp = (t >> 5) * 32 + lane / lpl;  // group id within the warp
  // cheap 32-bit hash (a few IMADs): the address math must not be the limit
  uint32_t h = (uint32_t)grp * 0x9E3779B1u ^ ((uint32_t)j + (uint32_t)seed) * 0x85EBCA77u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  const uint32_t line = (uint32_t)h & (mask >> 5);
  // distinct slots for the lanes sharing a line; a random slot otherwise
  // (spreads shared-memory banks like a real vertex-id access)
  const uint32_t span = 32u / (uint32_t)lpl;
  return (line << 5) | ((lane % lpl) * span + (h >> 27) % span);
}

template <int K, int F>
__global__ void sweep_kernel(uint32_t *buf, uint32_t mask, int iters, int lpl, uint64_t seed,
                             unsigned long long *sink) {
  extern __shared__ uint32_t sm[];
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (K >= kSmemLoad) {
    for (uint32_t i = threadIdx.x; i <= mask; i += blockDim.x) sm[i] = 0xFFFFFFFFu - i;
    __syncthreads();
  }
  uint32_t acc = 0;
  for (int it = 0; it < iters; it++) {
    uint32_t idx[F];
#pragma unroll
    for (int j = 0; j < F; j++) idx[j] = slot_of(seed, t, (uint64_t)it * F + j, mask, lpl);
    if (K == kGlobalLoad) {
      uint32_t v[F];
#pragma unroll
      for (int j = 0; j < F; j++) v[j] = buf[idx[j]];
#pragma unroll
      for (int j = 0; j < F; j++) acc += v[j];
    } else if (K == kGlobalRedMin) {
#pragma unroll
      for (int j = 0; j < F; j++)
        asm volatile("red.relaxed.gpu.global.min.u32 [%0], %1;" ::"l"(buf + idx[j]), "r"(idx[j] ^ (uint32_t)it)
                     : "memory");
    } else if (K == kSmemLoad) {
      uint32_t v[F];
#pragma unroll
      for (int j = 0; j < F; j++) v[j] = sm[idx[j]];
#pragma unroll
      for (int j = 0; j < F; j++) acc += v[j];
    } else if (K == kSmemAtomMin) {
#pragma unroll
      for (int j = 0; j < F; j++) atomicMin(sm + idx[j], idx[j] ^ (uint32_t)it);
    } else {  // read filter, then atomicMin only when it would improve
      uint32_t v[F];
#pragma unroll
      for (int j = 0; j < F; j++) v[j] = sm[idx[j]];
#pragma unroll
      for (int j = 0; j < F; j++) {
        const uint32_t m = (idx[j] * 2654435761u) ^ (uint32_t)it;
        if (m < v[j]) atomicMin(sm + idx[j], m);
      }
    }
  }
  if (K >= kSmemLoad) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i <= mask; i += blockDim.x) acc += sm[i];
  }
  if (acc == 0x12345u) atomicAdd(sink, 1ull);
}

template <int K, int F>
float run(uint32_t *buf, uint32_t mask, int grid, int block, int iters, int lpl, size_t smem,
          unsigned long long *sink) {
  auto kern = sweep_kernel<K, F>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms = 0.f;
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(a);
    kern<<<grid, block, smem>>>(buf, mask, iters, lpl, 1234567ull + rep, sink);
    cudaEventRecord(b);
  }
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return -1.f;
  }
  return ms;
}

template <int K>
float run_f(int F, uint32_t *buf, uint32_t mask, int grid, int block, int iters, int lpl,
            size_t smem, unsigned long long *sink) {
  switch (F) {
    case 1: return run<K, 1>(buf, mask, grid, block, iters, lpl, smem, sink);
    case 2: return run<K, 2>(buf, mask, grid, block, iters, lpl, smem, sink);
    case 4: return run<K, 4>(buf, mask, grid, block, iters, lpl, smem, sink);
    case 8: return run<K, 8>(buf, mask, grid, block, iters, lpl, smem, sink);
    default: return run<K, 16>(buf, mask, grid, block, iters, lpl, smem, sink);
  }
}

static const char *kNames[] = {"global_load_u32", "global_red_min_u32", "smem_load_u32",
                               "smem_atomic_min_u32", "smem_filter_then_atomic_min"};

void point(int K, int F, size_t bytes, int ctas_per_sm, int block, int lpl, uint32_t *buf,
           unsigned long long *sink, int sms, int clk_mhz) {
  const uint32_t mask = (uint32_t)(bytes / 4 - 1);
  const int grid = sms * ctas_per_sm;
  const double threads = (double)grid * block;
  const int iters = (int)((double)(1ull << 30) / (threads * F)) + 1;
  const size_t smem = K >= kSmemLoad ? bytes : 0;
  float ms = -1.f;
  switch (K) {
    case 0: ms = run_f<0>(F, buf, mask, grid, block, iters, lpl, smem, sink); break;
    case 1: ms = run_f<1>(F, buf, mask, grid, block, iters, lpl, smem, sink); break;
    case 2: ms = run_f<2>(F, buf, mask, grid, block, iters, lpl, smem, sink); break;
    case 3: ms = run_f<3>(F, buf, mask, grid, block, iters, lpl, smem, sink); break;
    default: ms = run_f<4>(F, buf, mask, grid, block, iters, lpl, smem, sink); break;
  }
  if (ms <= 0.f) return;
  const double ops = threads * F * iters;
  const double gops = ops / (ms * 1e-3) / 1e9;
  const double lines = gops / lpl;  // distinct 128-byte lines per second (G)
  printf("{\"kind\": \"%s\", \"bytes\": %zu, \"in_flight\": %d, \"ctas_per_sm\": %d, \"block\": %d, "
         "\"threads_per_sm\": %d, \"lanes_per_line\": %d, \"G_access_per_s\": %.1f, "
         "\"G_lines_per_s\": %.1f, \"lines_per_sm_clk\": %.3f, \"access_per_sm_clk\": %.3f}\n",
         kNames[K], bytes, F, ctas_per_sm, block, ctas_per_sm * block, lpl, gops, lines,
         lines * 1e9 / (sms * (double)clk_mhz * 1e6), gops * 1e9 / (sms * (double)clk_mhz * 1e6));
  fflush(stdout);
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  const int clk = clk_khz / 1000;
  uint32_t *buf = nullptr;
  unsigned long long *sink = nullptr;
  cudaMalloc(&buf, 1ull << 30);
  cudaMemset(buf, 0xFF, 1ull << 30);
  cudaMalloc(&sink, 8);
  // 1. in-flight x occupancy, L2-resident random loads, one line per lane
  for (int F : {1, 2, 4, 8, 16})
    for (int cps : {1, 2, 4, 8}) point(kGlobalLoad, F, 16u << 20, cps, 256, 1, buf, sink, sms, clk);
  // 2. array size (L1 / L2 / HBM) at the best occupancy
  for (size_t bytes : {(size_t)64 << 10, (size_t)16 << 20, (size_t)256 << 20, (size_t)1 << 30})
    point(kGlobalLoad, 8, bytes, 8, 256, 1, buf, sink, sms, clk);
  // 3. lanes per line: wavefront (line) rate vs access rate
  for (int lpl : {1, 2, 4, 8, 16, 32}) {
    point(kGlobalLoad, 8, 16u << 20, 8, 256, lpl, buf, sink, sms, clk);
    point(kGlobalLoad, 8, 64u << 10, 8, 256, lpl, buf, sink, sms, clk);
  }
  // 4. reductions
  for (int F : {4, 8}) point(kGlobalRedMin, F, 16u << 20, 8, 256, 1, buf, sink, sms, clk);
  // 5. shared memory: random loads / atomics on a per-CTA table
  for (int K : {kSmemLoad, kSmemAtomMin, kSmemFilterMin})
    for (size_t bytes : {(size_t)32 << 10, (size_t)96 << 10})
      for (int F : {4, 8}) point(K, F, bytes, bytes > (64 << 10) ? 2 : 4, 512, 1, buf, sink, sms, clk);
  cudaFree(buf);
  return 0;
}
