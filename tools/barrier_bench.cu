// barrier_bench.cu -- cost of one grid barrier of the persistent kernels
// (148 CTAs x 1024 threads, co-resident), by variant:
//   0  shipped kArriveRed: bar.sync; fence; red.release.add; spin ld.acquire; fence; bar.sync
//   1  no fences (release / acquire carry the ordering)
//   2  fence after the spin only
//   3  kArriveAtomic: atomicAdd with return, last arriver bumps gen
// Also: one barrier + a global counter read by every thread (the pattern
// after each superstep) vs the counter read by thread 0 into shared memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bb tools/barrier_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

struct Bar { unsigned count, gen; };

__device__ __forceinline__ unsigned ld_acq(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int V>
__device__ __forceinline__ void gsync(Bar *b, unsigned &gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (V == 3) {
      __threadfence();
      const unsigned arrived = atomicAdd(&b->count, 1u);
      if (arrived == gridDim.x - 1) {
        b->count = 0;
        __threadfence();
        atomicExch(&b->gen, gen + 1);
      } else {
        while (ld_acq(&b->gen) == gen) {}
      }
      __threadfence();
    } else {
      if (V == 0) __threadfence();
      const unsigned target = (gen + 1) * gridDim.x;
      asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(&b->count), "r"(1u) : "memory");
      while ((int)(ld_acq(&b->count) - target) < 0) {}
      if (V == 0 || V == 2) __threadfence();
    }
  }
  gen++;
  __syncthreads();
}

template <int V>
__global__ void __launch_bounds__(1024, 1) kern(Bar *b, int iters, unsigned long long *ctr, int mode,
                                              unsigned *sink) {
  __shared__ unsigned long long s_v;
  unsigned gen = 0;
  unsigned acc = 0;
  for (int i = 0; i < iters; i++) {
    gsync<V>(b, gen);
    if (mode == 1) {
      acc += (unsigned)ctr[i & 7];
    } else if (mode == 2) {
      if (threadIdx.x == 0) s_v = ctr[i & 7];
      __syncthreads();
      acc += (unsigned)s_v;
    }
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

template <int V>
float run(int grid, int iters, int mode, Bar *b, unsigned long long *ctr, unsigned *sink) {
  cudaMemset(b, 0, sizeof(Bar));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  void *args[] = {&b, &iters, &ctr, &mode, &sink};
  cudaLaunchCooperativeKernel((void *)kern<V>, grid, 1024, args, 0, 0);  // warm-up
  cudaDeviceSynchronize();
  cudaMemset(b, 0, sizeof(Bar));
  cudaEventRecord(e0);
  cudaLaunchCooperativeKernel((void *)kern<V>, grid, 1024, args, 0, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms * 1000.f / iters;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  Bar *b;
  unsigned long long *ctr;
  unsigned *sink;
  cudaMalloc(&b, 64);
  cudaMalloc(&ctr, 64);
  cudaMemset(ctr, 0, 64);
  cudaMalloc(&sink, 4);
  const int iters = 20000;
  for (int grid : {sms, sms / 2, 32}) {
    printf("grid %d: us per barrier  shipped %.3f  no-fence %.3f  fence-after %.3f  atomic %.3f\n",
           grid, run<0>(grid, iters, 0, b, ctr, sink), run<1>(grid, iters, 0, b, ctr, sink),
           run<2>(grid, iters, 0, b, ctr, sink), run<3>(grid, iters, 0, b, ctr, sink));
    printf("grid %d: barrier + counter read: every thread %.3f  thread 0 -> smem %.3f (shipped barrier)\n",
           grid, run<0>(grid, iters, 1, b, ctr, sink), run<0>(grid, iters, 2, b, ctr, sink));
  }
  return 0;
}
