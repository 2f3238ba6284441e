// FP64 tensor-core (mma.sync f64) throughput on B200 for the shapes PTX offers on sm_100a,
// vs plain DFMA: decides how the separable grid path's LSE convolutions are computed.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                         \
  do {                                                                \
    cudaError_t e = (x);                                              \
    if (e != cudaSuccess) {                                           \
      printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);     \
      exit(1);                                                        \
    }                                                                 \
  } while (0)

template <int SHAPE>
__global__ void k_mma(double* out, int iters) {
  // 8 independent accumulator sets per warp
  double c[8][4];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  double a[4], b[2];
  for (int j = 0; j < 4; ++j) a[j] = 1e-3 * (threadIdx.x + j);
  b[0] = 0.5; b[1] = 0.25;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (SHAPE == 0) {  // m8n8k4: 256 FMA
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a[0]), "d"(b[0]));
      } else if (SHAPE == 1) {  // m16n8k4: 512 FMA
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5}, {%6}, {%0, %1, %2, %3};"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      } else if (SHAPE == 2) {  // m16n8k8: 1024 FMA
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      }
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 1234.5) out[0] = s;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 64));
  const int iters = 4000;
  const double fma_per[3] = {256, 512, 1024};
  const char* names[3] = {"m8n8k4", "m16n8k4", "m16n8k8"};
  for (int shape = 0; shape < 3; ++shape) {
    for (int warps : {4, 8, 16}) {
      cudaEvent_t e0, e1;
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      auto run = [&]() {
        if (shape == 0) k_mma<0><<<sms, 32 * warps>>>(out, iters);
        else if (shape == 1) k_mma<1><<<sms, 32 * warps>>>(out, iters);
        else k_mma<2><<<sms, 32 * warps>>>(out, iters);
      };
      run();
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      run();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double fmas = fma_per[shape] * 8.0 * iters * warps * sms;
      printf("{\"shape\": \"%s\", \"warps_per_sm\": %d, \"tflops\": %.2f}\n", names[shape], warps,
             2 * fmas / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
