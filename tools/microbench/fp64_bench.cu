// Microbenchmarks that decide the DXG sweep design on B200 (sm_100a):
//  1. DFMA issue throughput (the FP64 roofline denominator),
//  2. table-driven FP64 exp (lane-replicated smem table) vs libdevice exp: accuracy + throughput,
//  3. HBM streaming read bandwidth with 16 B/lane loads.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

template <int LOGN>
struct ExpTab {
  static constexpr int N = 1 << LOGN;
};

// table-driven exp(x - m*ln2/N): returns value, integer shift applied in the exponent
template <int LOGN>
__device__ __forceinline__ double texp(double x, int m, const double* __restrict__ tab_lane) {
  constexpr int N = 1 << LOGN;
  const double K = (double)N / 0.69314718055994530942;
  const double L = 0.69314718055994530942 / (double)N;
  const double MAGIC = 6755399441055744.0;  // 1.5 * 2^52
  double t = fma(x, K, MAGIC);
  int k = __double2loint(t);
  double kd = t - MAGIC;
  double r = fma(kd, -L, x);
  int kk = max(k - m, -1000 * N);
  int idx = kk & (N - 1);
  int e = kk >> LOGN;
  double T = tab_lane[idx * 16];
  T = __hiloint2double(__double2hiint(T) + (e << 20), __double2loint(T));
  double p;
  if (LOGN >= 8) {
    p = fma(fma(fma(1.0 / 24, r, 1.0 / 6), r, 0.5), r, 1.0);
  } else {
    p = fma(fma(fma(fma(1.0 / 120, r, 1.0 / 24), r, 1.0 / 6), r, 0.5), r, 1.0);
  }
  double ep = fma(r, p, 1.0);
  return T * ep;
}

template <int LOGN>
__device__ void fill_table(double* tab) {
  constexpr int N = 1 << LOGN;
  for (int i = threadIdx.x; i < N * 16; i += blockDim.x) {
    int j = i / 16;
    tab[i] = exp2((double)j / N);
  }
  __syncthreads();
}

// accuracy: compute texp for given x array, write result
template <int LOGN>
__global__ void texp_eval(const double* x, double* y, int n) {
  extern __shared__ double tab[];
  fill_table<LOGN>(tab);
  const double* tl = tab + (threadIdx.x & 15);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[i] = texp<LOGN>(x[i], 0, tl);
}

__global__ void libexp_eval(const double* x, double* y, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = exp(x[i]);
}

// throughput: sum of exp(fma(-a, c, -b)) over a register-generated stream (no memory)
template <int LOGN>
__global__ void texp_tput(double* out, int iters, double a) {
  extern __shared__ double tab[];
  fill_table<LOGN>(tab);
  const double* tl = tab + (threadIdx.x & 15);
  double c0 = (threadIdx.x & 31) * (1.0 / 37.0), c1 = c0 + 0.11, c2 = c0 + 0.23, c3 = c0 + 0.37;
  double b0 = -0.5, s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < iters; ++i) {
    s0 += texp<LOGN>(fma(-a, c0, b0), 0, tl);
    s1 += texp<LOGN>(fma(-a, c1, b0), 0, tl);
    s2 += texp<LOGN>(fma(-a, c2, b0), 0, tl);
    s3 += texp<LOGN>(fma(-a, c3, b0), 0, tl);
    c0 += 1e-3; c1 += 1e-3; c2 += 1e-3; c3 += 1e-3;
  }
  double s = s0 + s1 + s2 + s3;
  if (s == 12345.678) out[0] = s;
}

__global__ void libexp_tput(double* out, int iters, double a) {
  double c0 = (threadIdx.x & 31) * (1.0 / 37.0), c1 = c0 + 0.11, c2 = c0 + 0.23, c3 = c0 + 0.37;
  double b0 = -0.5, s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < iters; ++i) {
    s0 += exp(fma(-a, c0, b0));
    s1 += exp(fma(-a, c1, b0));
    s2 += exp(fma(-a, c2, b0));
    s3 += exp(fma(-a, c3, b0));
    c0 += 1e-3; c1 += 1e-3; c2 += 1e-3; c3 += 1e-3;
  }
  double s = s0 + s1 + s2 + s3;
  if (s == 12345.678) out[0] = s;
}


// Variant A: same FP64 op count as texp (10), no integer ops / no table
__global__ void polyonly_tput(double* out, int iters, double a) {
  double c0 = (threadIdx.x & 31) * (1.0 / 37.0), c1 = c0 + 0.11, c2 = c0 + 0.23, c3 = c0 + 0.37;
  double b0 = -0.5, s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  const double K = 369.32993046757470, L = 0.0027076061740622864, M = 6755399441055744.0;
#define PO(c, s) { double x = fma(-a, c, b0); double t = fma(x, K, M); double kd = t - M; double r = fma(kd, -L, x); \
    double p = fma(fma(fma(1.0/24, r, 1.0/6), r, 0.5), r, 1.0); s = fma(t, fma(r, p, 1.0), s); }
  for (int i = 0; i < iters; ++i) {
    PO(c0, s0) PO(c1, s1) PO(c2, s2) PO(c3, s3)
    c0 += 1e-3; c1 += 1e-3; c2 += 1e-3; c3 += 1e-3;
  }
  double s = s0 + s1 + s2 + s3;
  if (s == 12345.678) out[0] = s;
}
// Variant B: texp without clamp and with table index only (no exponent scaling)
__global__ void texp_noclamp_tput(double* out, int iters, double a) {
  extern __shared__ double tab[];
  fill_table<8>(tab);
  const double* tl = tab + (threadIdx.x & 15);
  double c0 = (threadIdx.x & 31) * (1.0 / 37.0), c1 = c0 + 0.11, c2 = c0 + 0.23, c3 = c0 + 0.37;
  double b0 = -0.5, s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  const double K = 369.32993046757470, L = 0.0027076061740622864, M = 6755399441055744.0;
#define PB(c, s) { double x = fma(-a, c, b0); double t = fma(x, K, M); double kd = t - M; double r = fma(kd, -L, x); \
    int k = __double2loint(t); double T = tl[(k & 255) * 16]; \
    double p = fma(fma(fma(1.0/24, r, 1.0/6), r, 0.5), r, 1.0); s = fma(T, fma(r, p, 1.0), s); }
  for (int i = 0; i < iters; ++i) {
    PB(c0, s0) PB(c1, s1) PB(c2, s2) PB(c3, s3)
    c0 += 1e-3; c1 += 1e-3; c2 += 1e-3; c3 += 1e-3;
  }
  double s = s0 + s1 + s2 + s3;
  if (s == 12345.678) out[0] = s;
}

__global__ void stream_read(const double2* __restrict__ p, size_t n2, double* out) {
  double s = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 v0 = __ldcs(p + i), v1 = __ldcs(p + i + stride), v2 = __ldcs(p + i + 2 * stride), v3 = __ldcs(p + i + 3 * stride);
    s += v0.x + v0.y + v1.x + v1.y + v2.x + v2.y + v3.x + v3.y;
  }
  for (; i < n2; i += stride) { double2 v = p[i]; s += v.x + v.y; }
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("device %s sms %d clock %d kHz\n", prop.name, sms, prop.clockRate);
  double* dout; CK(cudaMalloc(&dout, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // 1. DFMA
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    int iters = 4000;
    dfma_kernel<<<blocks, tpb>>>(dout, 10, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int rep = 0; rep < 5; ++rep) dfma_kernel<<<blocks, tpb>>>(dout, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double dfma = 5.0 * blocks * tpb * (double)iters * 64;
    printf("DFMA tpb %d: %.3f T DFMA/s (%.2f TFLOPS) = %.1f DFMA/clk/SM at %d MHz\n", tpb, dfma / (ms * 1e-3) / 1e12,
           2 * dfma / (ms * 1e-3) / 1e12, dfma / (ms * 1e-3) / (sms * prop.clockRate * 1e3), prop.clockRate / 1000);
  }
  // 2. exp accuracy
  const int NX = 1 << 22;
  std::vector<double> hx(NX), hy(NX), hl(NX);
  srand(1);
  for (int i = 0; i < NX; ++i) hx[i] = -745.0 + 760.0 * (rand() / (double)RAND_MAX);
  double *dx, *dy; CK(cudaMalloc(&dx, NX * 8)); CK(cudaMalloc(&dy, NX * 8));
  CK(cudaMemcpy(dx, hx.data(), NX * 8, cudaMemcpyHostToDevice));
  libexp_eval<<<1024, 256>>>(dx, dy, NX); CK(cudaMemcpy(hl.data(), dy, NX * 8, cudaMemcpyDeviceToHost));
  auto check = [&](const char* name) {
    double maxrel = 0; long worst_i = -1;
    for (int i = 0; i < NX; ++i) {
      double ref = std::exp(hx[i]);
      if (ref < 1e-300) continue;
      double rel = std::fabs(hy[i] - ref) / ref;
      if (rel > maxrel) { maxrel = rel; worst_i = i; }
    }
    printf("%s max rel err vs host exp: %.3e (x=%.6f)\n", name, maxrel, worst_i >= 0 ? hx[worst_i] : 0.0);
  };
  hy = hl; check("libdevice exp");
  texp_eval<6><<<1024, 256, 64 * 16 * 8>>>(dx, dy, NX); CK(cudaMemcpy(hy.data(), dy, NX * 8, cudaMemcpyDeviceToHost)); check("texp N=64 deg5");
  CK(cudaFuncSetAttribute(texp_eval<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 16 * 8));
  texp_eval<8><<<1024, 256, 256 * 16 * 8>>>(dx, dy, NX); CK(cudaMemcpy(hy.data(), dy, NX * 8, cudaMemcpyDeviceToHost)); check("texp N=256 deg4");
  // 3. exp throughput
  {
    int tpb = 256, blocks = sms * 8, iters = 2000;
    libexp_tput<<<blocks, tpb>>>(dout, 10, 3.0); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); libexp_tput<<<blocks, tpb>>>(dout, iters, 3.0); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double ne = 4.0 * blocks * tpb * iters;
    printf("libdevice exp: %.1f G exp/s (%.2f exp/clk/SM)\n", ne / (ms * 1e-3) / 1e9, ne / (ms * 1e-3) / (sms * prop.clockRate * 1e3));
    texp_tput<6><<<blocks, tpb, 64 * 16 * 8>>>(dout, 10, 3.0); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); texp_tput<6><<<blocks, tpb, 64 * 16 * 8>>>(dout, iters, 3.0); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("texp N=64: %.1f G exp/s (%.2f exp/clk/SM)\n", ne / (ms * 1e-3) / 1e9, ne / (ms * 1e-3) / (sms * prop.clockRate * 1e3));
    CK(cudaFuncSetAttribute(texp_tput<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 16 * 8));
    texp_tput<8><<<blocks, tpb, 256 * 16 * 8>>>(dout, 10, 3.0); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); texp_tput<8><<<blocks, tpb, 256 * 16 * 8>>>(dout, iters, 3.0); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("texp N=256: %.1f G exp/s (%.2f exp/clk/SM)\n", ne / (ms * 1e-3) / 1e9, ne / (ms * 1e-3) / (sms * prop.clockRate * 1e3));
  }

  {
    int tpb = 256, blocks = sms * 6, iters = 2000;
    double ne = 4.0 * blocks * tpb * iters;
    polyonly_tput<<<blocks, tpb>>>(dout, 10, 3.0); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); polyonly_tput<<<blocks, tpb>>>(dout, iters, 3.0); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("polyonly (10 FP64, no int): %.2f exp/clk/SM\n", ne / (ms * 1e-3) / (sms * prop.clockRate * 1e3));
    CK(cudaFuncSetAttribute(texp_noclamp_tput, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 16 * 8));
    texp_noclamp_tput<<<blocks, tpb, 256 * 16 * 8>>>(dout, 10, 3.0); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); texp_noclamp_tput<<<blocks, tpb, 256 * 16 * 8>>>(dout, iters, 3.0); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("texp table-only (no clamp/scale): %.2f exp/clk/SM\n", ne / (ms * 1e-3) / (sms * prop.clockRate * 1e3));
  }
  // 4. HBM read
  {
    size_t bytes = (size_t)8 << 30;
    double2* p; CK(cudaMalloc(&p, bytes)); CK(cudaMemset(p, 0, bytes));
    size_t n2 = bytes / 16;
    for (int bpsm : {4, 8, 16}) {
      int blocks = sms * bpsm;
      stream_read<<<blocks, 256>>>(p, n2, dout); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      for (int rep = 0; rep < 5; ++rep) stream_read<<<blocks, 256>>>(p, n2, dout);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("stream read %d blocks/SM: %.1f GB/s\n", bpsm, 5.0 * bytes / (ms * 1e-3) / 1e9);
    }
    cudaFree(p);
  }
  return 0;
}
