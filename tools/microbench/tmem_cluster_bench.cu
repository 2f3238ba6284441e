// TMEM ld/st throughput (tcgen05.ld/st 32x32b) and co-resident cluster capacity on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1;} } while (0)

__global__ void __launch_bounds__(512, 1) tmem_bw(unsigned* out, int iters) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s;
  // 16 warps: 4 per lane quarter, each gets 128 columns
  const uint32_t ta = base + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
  uint32_t v[32];
  for (int i = 0; i < 32; ++i) v[i] = threadIdx.x * 7 + i;
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                 :: "r"(ta + (it & 3) * 32), "r"(v[0]),"r"(v[1]),"r"(v[2]),"r"(v[3]),"r"(v[4]),"r"(v[5]),"r"(v[6]),"r"(v[7]),"r"(v[8]),"r"(v[9]),"r"(v[10]),"r"(v[11]),"r"(v[12]),"r"(v[13]),"r"(v[14]),"r"(v[15]),"r"(v[16]),"r"(v[17]),"r"(v[18]),"r"(v[19]),"r"(v[20]),"r"(v[21]),"r"(v[22]),"r"(v[23]),"r"(v[24]),"r"(v[25]),"r"(v[26]),"r"(v[27]),"r"(v[28]),"r"(v[29]),"r"(v[30]),"r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
                 : "r"(ta + ((it + 1) & 3) * 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    v[it & 31] += 1;
  }
  for (int i = 0; i < 32; ++i) acc += v[i];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(base));
  if (acc == 12345) out[0] = acc;
}

__global__ void cluster_probe(int* out) {
  if (threadIdx.x == 0) atomicAdd(out, 1);
}

int main() {
  unsigned* d; CK(cudaMalloc(&d, 64));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  tmem_bw<<<sms, 512>>>(d, 10); CK(cudaDeviceSynchronize());
  int iters = 20000;
  cudaEventRecord(e0); tmem_bw<<<sms, 512>>>(d, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double bytes = 2.0 * sms * 512.0 * 32 * 4 * iters;  // st + ld, 32 x 32-bit per thread
  printf("TMEM st+ld: %.1f TB/s total, %.1f B/clk/SM (at %d MHz)\n", bytes / (ms * 1e-3) / 1e12,
         bytes / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs * 64); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 160 * 1024;
    cfg.attrs = at; cfg.numAttrs = 1;
    if (cs > 8) cudaFuncSetAttribute(cluster_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(cluster_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    int nc = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, cluster_probe, &cfg);
    printf("cluster size %2d: max active clusters %d (%d SMs) %s\n", cs, nc, nc * cs, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
