// Shared device code for the DXG sweeps on sm_100a.
//
// Numerics: every row softmax of the implicit plan
//   p_ij = exp(x_ij - L_i),  x_ij = -(a C_ij + b_j)        (dxg.py:199-203)
// is evaluated with a table-driven FP64 exp whose row shift is an INTEGER in
// units of ln2/512:  exp(x - m*ln2/512) = 2^((k-m)/512) * exp(r),
//   k = round(x*512/ln2),  r = x - k*ln2/512,  |r| <= ln2/1024.
// 2^(j/512) comes from a lane-replicated shared-memory table (conflict-free
// LDS.64), the 2^e scaling is an integer add on the exponent field, and exp(r)
// is a degree-3 minimax polynomial (max rel. error 1.1e-15).  Per element and
// weight set this is 8 FP64 instructions + 6 integer/LDS instructions, versus
// 16 FP64 for libdevice exp: on sm_100a an FP64 instruction occupies the
// dispatch port for 2 cycles, so the integer work is not free and is kept
// minimal (profiles/r01_microbench.md).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/leanot_b200.h"

namespace leanot {

constexpr int LOGN = 9;
constexpr int NTAB = 1 << LOGN;
constexpr int TAB_LANES = 16;
constexpr int TAB_BYTES = NTAB * TAB_LANES * 8;  // 64 KB
constexpr double LN2 = 0.693147180559945309417232121458;
constexpr double KINV = NTAB / LN2;   // 512/ln2 (rounding only moves the nearest-k choice)
constexpr double LSTEP = LN2 / NTAB;  // ln2/512, exact division of the double ln2
constexpr double MAGIC = 6755399441055744.0;      // 1.5 * 2^52
constexpr int KLO = -1000 * NTAB;                 // exp(x-s) < 2^-1000 is flushed to ~2^-1000
// minimax exp(r) on |r| <= ln2/1024 (relative error <= 1.1e-15), see DESIGN.md §3
constexpr double EC0 = 0.9999999999999989;
constexpr double EC1 = 1.0000000000000024;
constexpr double EC2 = 0.5000000190914873;
constexpr double EC3 = 0.16666666285067583;

// The same coefficients in the constant bank: a DFMA takes one constant-bank operand
// directly, so the hot loops do not re-materialize 64-bit immediates per stage.
__constant__ double c_lstep = LSTEP;
__constant__ double c_ec0 = EC0, c_ec1 = EC1, c_ec3 = EC3;

// Biased table: entry j holds 2^(j/512) (correctly rounded) with (j << 11) subtracted
// from its high word.  For kk = 512 e + j the scaled value 2^(kk/512) then has
// high word  hi(T'[j]) + (kk << 11)  -- one LEA, no masking -- because
// kk << 11 = (e << 20) + (j << 11).  Filled by the host at library init.  The
// library is one translation unit (leanot_lib.cu includes every .cu file), so
// this definition exists exactly once.
__device__ double g_exp2_table[NTAB];

// One global read per entry, replicated with 16-byte stores (entry j occupies the 128 B
// at smem_tab + 16 j: one copy per lane of a half-warp).
__device__ __forceinline__ void load_table(double* smem_tab) {
  for (int i = threadIdx.x; i < NTAB * (TAB_LANES / 2); i += blockDim.x) {
    const double v = g_exp2_table[i / (TAB_LANES / 2)];
    reinterpret_cast<double2*>(smem_tab)[i] = make_double2(v, v);
  }
}

// Shared-window address of this lane's replica of the table (base + lane*8), opaque
// to the compiler so it is kept in one register instead of being re-derived.
__device__ __forceinline__ uint32_t lane_tab_addr(const void* smem_tab) {
  uint32_t v = (uint32_t)__cvta_generic_to_shared(smem_tab) + ((threadIdx.x & 15u) << 3);
  asm volatile("" : "+r"(v));
  return v;
}

// Scaled table value 2^((k - m)/512) for t = fma(x, KINV, MAGIC); the low word of t
// holds k (mod 2^32), so the subtraction of the row shift is exact modular arithmetic.
// 4 integer instructions + 1 LDS: VIADDMNMX (shift+clamp), LOP3 (j = kk & 511),
// LEA (address), IMAD (exponent add, biased table).
__device__ __forceinline__ double tab_scaled(uint32_t tb, double t, uint32_t mlo) {
  const int kk = max((int)((uint32_t)__double2loint(t) - mlo), KLO);
  double T;
  asm("{\n\t.reg .b32 j, a;\n\tand.b32 j, %1, 511;\n\tmad.lo.u32 a, j, 128, %2;\n\t"
      "ld.shared.f64 %0, [a];\n\t}"
      : "=d"(T) : "r"(kk), "r"(tb));
  return __hiloint2double(__double2hiint(T) + (kk << 11), __double2loint(T));
}

// exp(x - m*LSTEP) (pass A form): returns T * poly(r)
__device__ __forceinline__ double texp(uint32_t tb, double x, uint32_t mlo) {
  const double t = fma(x, KINV, MAGIC);
  const double kd = t - MAGIC;
  const double r = fma(kd, -c_lstep, x);
  const double T = tab_scaled(tb, t, mlo);
  const double p = fma(fma(c_ec3, r, EC2), r, c_ec1);
  return T * fma(r, p, c_ec0);
}

// acc += exp(x - m*LSTEP)
__device__ __forceinline__ void texp_acc(uint32_t tb, double x, uint32_t mlo, double& acc) {
  const double t = fma(x, KINV, MAGIC);
  const double kd = t - MAGIC;
  const double r = fma(kd, -c_lstep, x);
  const double T = tab_scaled(tb, t, mlo);
  const double p = fma(fma(c_ec3, r, EC2), r, c_ec1);
  acc = fma(T, fma(r, p, c_ec0), acc);
}

// acc += g * exp(x - m*LSTEP) with g folded into the polynomial: gc = g*{EC0..EC3}
__device__ __forceinline__ void texp_gacc(uint32_t tb, double x, uint32_t mlo, double g0, double g1, double g2,
                                          double g3, double& acc) {
  const double t = fma(x, KINV, MAGIC);
  const double kd = t - MAGIC;
  const double r = fma(kd, -c_lstep, x);
  const double T = tab_scaled(tb, t, mlo);
  const double q = fma(fma(fma(g3, r, g2), r, g1), r, g0);
  acc = fma(T, q, acc);
}

// ---------------------------------------------------------------------------
// cost providers (core.py:200-288).  Normalized C_ij = raw_ij * inv_scale for
// on-the-fly kinds; the stored kind holds the normalized matrix already.
// ---------------------------------------------------------------------------

struct CostView {
  int kind, p, dim, height, width;
  int64_t n, ld, row_base;
  const double* mat;
  const double* feat;
  const double* gcoord;  // grid: [row(n) | col(n)] as doubles
  const double* norms;   // points, p = 2: |f_j|^2 (expanded-form sweeps), may be null
  double inv_scale;
};

__host__ __device__ inline CostView make_view(const leanot_cost_t& c) {
  CostView v;
  v.kind = c.kind; v.p = c.p; v.dim = c.dim; v.height = c.height; v.width = c.width;
  v.n = c.n; v.ld = c.ld; v.row_base = c.row_base; v.mat = c.mat; v.feat = c.feat;
  v.gcoord = c.grid_coords; v.norms = c.norms; v.inv_scale = c.inv_scale;
  return v;
}

__device__ __forceinline__ double ipow(double d, int p) {
  d = fabs(d);
  return p == 1 ? d : (p == 2 ? d * d : d * d * d);
}

// raw (un-normalized) on-the-fly cost between row features fi and column j
template <int DIM>
__device__ __forceinline__ double point_raw(const double* fi, const double* fj, int p) {
  double s;
  if (p == 2) {
    double d0 = fi[0] - fj[0];
    s = d0 * d0;
#pragma unroll
    for (int d = 1; d < DIM; ++d) { double dd = fi[d] - fj[d]; s = fma(dd, dd, s); }
  } else {
    s = ipow(fi[0] - fj[0], p);
#pragma unroll
    for (int d = 1; d < DIM; ++d) s += ipow(fi[d] - fj[d], p);
  }
  return s;
}

// ---------------------------------------------------------------------------
// reductions
// ---------------------------------------------------------------------------

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace leanot
