// Energy per instruction class on B200 under the 1 kW cap: each mode runs one
// instruction mix on every SM for a few seconds; tools/microbench/power_bench.sh samples
// SM clock and board power meanwhile.  Decides whether trading FP64 instructions for
// integer / shared-memory / FP32 ones makes the (power-capped) sweep faster.
//   dfma  8 independent DFMA chains per thread
//   ffma  8 independent FFMA chains per thread
//   int   IMAD / LOP3 / VIADDMNMX mix (the exp's integer part)
//   lds   conflict-free LDS.64 from a lane-replicated table
//   exp   the sweep's table exp (8 FP64 + 4 INT + 1 LDS) on register data
//   hbm   streaming 16 B/lane reads of a 16 GB buffer
//   l2    the same reads of a 48 MB buffer (L2-resident): separates DRAM from on-chip transport
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../paper_2511_11359_b200/csrc/leanot_common.cuh"

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

using namespace leanot;

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_ffma(double* out, int iters, float a, float b) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678f) out[0] = s;
}

__global__ void k_int(double* out, int iters, uint32_t m, uint32_t tb) {
  uint32_t x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 77u + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        int kk = max((int)(x[k] - m), KLO);
        uint32_t j = (uint32_t)kk & 511u;
        uint32_t ad = j * 128u + tb;
        x[k] = ad + ((uint32_t)kk << 11);
      }
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s ^= x[k];
  if (s == 12345u) out[0] = s;
}

__global__ void k_lds(double* out, int iters) {
  extern __shared__ __align__(16) char smem[];
  load_table(reinterpret_cast<double*>(smem));
  __syncthreads();
  const uint32_t tb = lane_tab_addr(smem);
  uint32_t idx[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) idx[k] = (threadIdx.x * 13u + k * 7u) & 511u;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double T;
      asm volatile("{\n\t.reg .b32 a;\n\tmad.lo.u32 a, %1, 128, %2;\n\tld.shared.f64 %0, [a];\n\t}"
                   : "=d"(T)
                   : "r"(idx[k]), "r"(tb));
      acc += __double2loint(T);
      idx[k] = (idx[k] + 37u + (acc & 1u)) & 511u;
    }
  if (acc == 12345u) out[0] = acc;
}

__global__ void k_exp(double* out, int iters, double na, double nb) {
  extern __shared__ __align__(16) char smem[];
  load_table(reinterpret_cast<double*>(smem));
  __syncthreads();
  const uint32_t tb = lane_tab_addr(smem);
  double c[8], acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    c[k] = (threadIdx.x * 8 + k) * (1.0 / 2048.0);
    acc[k] = 0.0;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) texp_acc(tb, fma(na, c[k], nb), 0u, acc[k]);
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = c[k] + 1e-9;  // keeps the loop honest (1 DADD / exp)
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_hbm(const uint4* __restrict__ p, int64_t n16, double* out) {
  uint32_t x = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i);
    x ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (x == 12345u) out[0] = x;
}

int main(int argc, char** argv) {
  const char* mode = argc > 1 ? argv[1] : "dfma";
  const double seconds = argc > 2 ? atof(argv[2]) : 3.0;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 64));
  // table for the smem modes (values irrelevant for power, but keep them finite)
  static double h_tab[NTAB];
  for (int j = 0; j < NTAB; ++j) h_tab[j] = 1.0 + j * 1e-3;
  CK(cudaMemcpyToSymbol(g_exp2_table, h_tab, sizeof(h_tab)));
  CK(cudaFuncSetAttribute(k_lds, cudaFuncAttributeMaxDynamicSharedMemorySize, TAB_BYTES));
  CK(cudaFuncSetAttribute(k_exp, cudaFuncAttributeMaxDynamicSharedMemorySize, TAB_BYTES));
  uint4* buf = nullptr;
  const int64_t bytes = 16LL << 30;
  const int64_t l2bytes = 48LL << 20;
  if (!strcmp(mode, "hbm")) CK(cudaMalloc(&buf, bytes));
  if (!strcmp(mode, "l2")) CK(cudaMalloc(&buf, l2bytes));
  const int blocks = sms * 2, threads = 512;
  const int iters = 20000;
  double ops_per_launch = 0;  // thread-level operations of the named class
  auto launch = [&]() {
    if (!strcmp(mode, "dfma")) { k_dfma<<<blocks, threads>>>(out, iters, 0.999, 1e-3); ops_per_launch = 64.0 * iters; }
    else if (!strcmp(mode, "ffma")) { k_ffma<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f); ops_per_launch = 64.0 * iters; }
    else if (!strcmp(mode, "int")) { k_int<<<blocks, threads>>>(out, iters, 3u, 0u); ops_per_launch = 16.0 * iters; }
    else if (!strcmp(mode, "lds")) { k_lds<<<blocks, threads, TAB_BYTES>>>(out, iters); ops_per_launch = 8.0 * iters; }
    else if (!strcmp(mode, "exp")) { k_exp<<<blocks, threads, TAB_BYTES>>>(out, iters / 4, -300.0, -1.0); ops_per_launch = 8.0 * iters / 4; }
    else if (!strcmp(mode, "hbm")) { k_hbm<<<sms * 4, 512>>>(buf, bytes / 16, out); ops_per_launch = (double)bytes / ((double)blocks * threads); }
    else if (!strcmp(mode, "l2")) {
      for (int rep = 0; rep < 64; ++rep) k_hbm<<<sms * 4, 512>>>(buf, l2bytes / 16, out);
      ops_per_launch = 64.0 * (double)l2bytes / ((double)blocks * threads);
    }
    else { printf("unknown mode\n"); exit(2); }
  };
  launch();
  CK(cudaDeviceSynchronize());
  auto t0 = std::chrono::steady_clock::now();
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  int launches = 0;
  while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < seconds) {
    for (int i = 0; i < 4; ++i, ++launches) launch();
    CK(cudaEventSynchronize(e0));
    CK(cudaDeviceSynchronize());
  }
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double total = ops_per_launch * (double)blocks * threads * launches;
  printf("{\"mode\": \"%s\", \"launches\": %d, \"seconds\": %.3f, \"ops_per_s\": %.4e}\n", mode, launches, ms / 1e3,
         total / (ms / 1e3));
  return 0;
}
