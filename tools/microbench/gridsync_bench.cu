// Cost of a grid-wide barrier on B200: cooperative_groups grid.sync() vs a hand-rolled
// sense-reversing barrier (one atomic per CTA + spin on a generation word).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* out) {
  cg::grid_group g = cg::this_grid();
  double v = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    v = v * 1.0000001 + 1e-9;
    g.sync();
  }
  if (v == 12345.0) out[0] = v;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ld_acquire(gen);
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      atomicExch(count, 0u);
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (ld_acquire(gen) == g) {
      }
    }
  }
  __syncthreads();
}

__global__ void k_own(int iters, double* out, unsigned* bar) {
  double v = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    v = v * 1.0000001 + 1e-9;
    grid_barrier(bar, bar + 32, gridDim.x);
  }
  if (v == 12345.0) out[0] = v;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  unsigned* bar;
  cudaMalloc(&out, 64);
  cudaMalloc(&bar, 256);
  cudaMemset(bar, 0, 256);
  for (int bps : {1, 2}) {
    const int G = sms * bps;
    int iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    void* a1[] = {&iters, &out};
    cudaLaunchCooperativeKernel((void*)k_cg, G, 256, a1, 0, 0);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k_cg, G, 256, a1, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"barrier\": \"cg grid.sync\", \"ctas\": %d, \"us_per_sync\": %.3f}\n", G, ms * 1e3 / iters);
    void* a2[] = {&iters, &out, &bar};
    cudaLaunchCooperativeKernel((void*)k_own, G, 256, a2, 0, 0);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k_own, G, 256, a2, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"barrier\": \"atomic+generation\", \"ctas\": %d, \"us_per_sync\": %.3f, \"err\": \"%s\"}\n", G,
           ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
