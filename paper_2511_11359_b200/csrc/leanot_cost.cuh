// Cost providers for the sweeps: one template per CostKernel kind (core.py:200-288).
// Each provider exposes
//   Row  row(i)                    per-row data (pointer or coordinates) in registers
//   Col  col(j)                    per-column data for the column pair (j, j+1)
//   void eval2(Row, Col, j, c0, c1) normalized C_ij, C_i,j+1
//   double eval1(Row, j)           single column (tails)
#pragma once
#include "leanot_common.cuh"

namespace leanot {

// ExplicitKernel: normalized matrix stored row-major in HBM (core.py:239-261)
struct CostStored {
  static constexpr bool kStored = true;
  static constexpr bool kGram = false;
  const double* mat;
  int64_t ld, row_base;
  struct Row { const double* p; };
  struct Col {};
  __device__ explicit CostStored(const CostView& v) : mat(v.mat), ld(v.ld), row_base(v.row_base) {}
  #ifdef LEANOT_DBG_WRAP
  __device__ __forceinline__ Row row(int64_t i) const { return Row{mat + ((i - row_base) % LEANOT_DBG_WRAP) * ld}; }
#else
  __device__ __forceinline__ Row row(int64_t i) const { return Row{mat + (i - row_base) * ld}; }
#endif
  __device__ __forceinline__ Col col(int64_t) const { return Col{}; }
  __device__ __forceinline__ void eval2(const Row& r, const Col&, int64_t j, double& c0, double& c1) const {
    double2 v = __ldg(reinterpret_cast<const double2*>(r.p + j));
    c0 = v.x; c1 = v.y;
  }
  // streaming variant for the column pass: evict-first, each row is read once per sweep
  __device__ __forceinline__ void eval2_stream(const Row& r, const Col&, int64_t j, double& c0, double& c1) const {
    double2 v = __ldcs(reinterpret_cast<const double2*>(r.p + j));
    c0 = v.x; c1 = v.y;
  }
  __device__ __forceinline__ double eval1(const Row& r, int64_t j) const { return __ldg(r.p + j); }
  // software-pipelined access: pre* issues the loads, get* consumes them
  template <int R> struct Pre2 { double2 v[R]; };
  template <int R>
  __device__ __forceinline__ void pre2(const Row (&rows)[R], const Col&, int64_t j, Pre2<R>& p) const {
#pragma unroll
    for (int r = 0; r < R; ++r) p.v[r] = __ldg(reinterpret_cast<const double2*>(rows[r].p + j));
  }
  template <int R>
  __device__ __forceinline__ void get2(const Row (&)[R], const Col&, const Pre2<R>& p, double (&c)[R][2]) const {
#pragma unroll
    for (int r = 0; r < R; ++r) { c[r][0] = p.v[r].x; c[r][1] = p.v[r].y; }
  }
  // four consecutive columns per thread as two 16-byte loads (j, j + 2).  Each load of a warp
  // uses half of every 32-byte sector it touches, but the second load hits the same sectors
  // in L1, so L2 traffic equals the algorithmic bytes (ncu lts__t_sectors_srcunit_tex_op_read
  // = 2.52e9 = 80 GB / 32 B).  A layout with whole-sector loads per instruction (pairs at 2t and
  // 2t + 512) removed the "excessive" L1 sectors but took 17 % more cycles (r02 A/B,
  // profiles/r02_colpass_layout.md), so it is not used.
  struct Pre4 { double2 v0, v1; };
  __device__ __forceinline__ void pre4(const Row& row, int64_t j, Pre4& p) const {
    p.v0 = __ldcs(reinterpret_cast<const double2*>(row.p + j));
    p.v1 = __ldcs(reinterpret_cast<const double2*>(row.p + j + 2));
  }
  // four consecutive columns (j % 4 == 0 not required; j even), for the column pass
  struct Col4 {};
  __device__ __forceinline__ Col4 col4(int64_t) const { return Col4{}; }
  __device__ __forceinline__ void eval4(const Row& r, const Col4&, int64_t j, double* c) const {
    double2 v0 = __ldcs(reinterpret_cast<const double2*>(r.p + j));
    double2 v1 = __ldcs(reinterpret_cast<const double2*>(r.p + j + 2));
    c[0] = v0.x; c[1] = v0.y; c[2] = v1.x; c[3] = v1.y;
  }
  __device__ __forceinline__ void get4(const Pre4& p, const Col4&, double* c) const {
    c[0] = p.v0.x; c[1] = p.v0.y; c[2] = p.v1.x; c[3] = p.v1.y;
  }
};

// Features of columns j, j+1 (j even, j + 1 < n) for the pass-A pipeline: the 2*DIM doubles
// are contiguous and 16-byte aligned (row-major features; validate_cost requires a 16-byte
// aligned base), so they arrive as DIM 16-byte loads instead of 2*DIM 8-byte ones.
template <int DIM>
__device__ __forceinline__ void col_pair(const double* f, int64_t j, double (&v0)[DIM], double (&v1)[DIM]) {
  const double2* q = reinterpret_cast<const double2*>(f + j * DIM);
  double e[2 * DIM];
#pragma unroll
  for (int t = 0; t < DIM; ++t) {
    const double2 w = __ldg(q + t);
    e[2 * t] = w.x;
    e[2 * t + 1] = w.y;
  }
#pragma unroll
  for (int d = 0; d < DIM; ++d) { v0[d] = e[d]; v1[d] = e[DIM + d]; }
}

// ColorKernel: sum_d |f_id - f_jd|^P / scale (core.py:264-288)
template <int DIM, int P>
struct CostPoints {
  static constexpr bool kStored = false;
  static constexpr bool kGram = false;
  const double* f;
  double inv;
  int64_t n;
  struct Row { double v[DIM]; };
  struct Col { double v0[DIM], v1[DIM]; };
  __device__ explicit CostPoints(const CostView& v) : f(v.feat), inv(v.inv_scale), n(v.n) {}
  __device__ __forceinline__ Row row(int64_t i) const {
    Row r;
#pragma unroll
    for (int d = 0; d < DIM; ++d) r.v[d] = __ldg(f + i * DIM + d);
    return r;
  }
  __device__ __forceinline__ Col col(int64_t j) const {
    Col c;
    int64_t j1 = j + 1 < n ? j + 1 : j;
#pragma unroll
    for (int d = 0; d < DIM; ++d) { c.v0[d] = __ldg(f + j * DIM + d); c.v1[d] = __ldg(f + j1 * DIM + d); }
    return c;
  }
  __device__ __forceinline__ static double raw(const double* a, const double* b) {
    double s;
    if (P == 2) {
      double d0 = a[0] - b[0];
      s = d0 * d0;
#pragma unroll
      for (int d = 1; d < DIM; ++d) { double dd = a[d] - b[d]; s = fma(dd, dd, s); }
    } else {
      double d0 = fabs(a[0] - b[0]);
      s = P == 1 ? d0 : d0 * d0 * d0;
#pragma unroll
      for (int d = 1; d < DIM; ++d) {
        double dd = fabs(a[d] - b[d]);
        s += P == 1 ? dd : dd * dd * dd;
      }
    }
    return s;
  }
  __device__ __forceinline__ void eval2(const Row& r, const Col& c, int64_t, double& c0, double& c1) const {
    c0 = raw(r.v, c.v0) * inv;
    c1 = raw(r.v, c.v1) * inv;
  }
  __device__ __forceinline__ void eval2_stream(const Row& r, const Col& c, int64_t j, double& c0, double& c1) const {
    eval2(r, c, j, c0, c1);
  }
  __device__ __forceinline__ double eval1(const Row& r, int64_t j) const {
    double b[DIM];
#pragma unroll
    for (int d = 0; d < DIM; ++d) b[d] = __ldg(f + j * DIM + d);
    return raw(r.v, b) * inv;
  }
  template <int R> struct Pre2 { Col c; };
  template <int R>
  __device__ __forceinline__ void pre2(const Row (&)[R], const Col&, int64_t j, Pre2<R>& p) const {
    col_pair<DIM>(f, j, p.c.v0, p.c.v1);
  }
  template <int R>
  __device__ __forceinline__ void get2(const Row (&rows)[R], const Col&, const Pre2<R>& p, double (&c)[R][2]) const {
#pragma unroll
    for (int r = 0; r < R; ++r) { c[r][0] = raw(rows[r].v, p.c.v0) * inv; c[r][1] = raw(rows[r].v, p.c.v1) * inv; }
  }
  struct Pre4 { Row r; };
  __device__ __forceinline__ void pre4(const Row& row, int64_t, Pre4& p) const { p.r = row; }
  struct Col4 { double v[4][DIM]; };
  __device__ __forceinline__ Col4 col4(int64_t j) const {
    Col4 c;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int64_t jj = j + q < n ? j + q : n - 1;
#pragma unroll
      for (int d = 0; d < DIM; ++d) c.v[q][d] = __ldg(f + jj * DIM + d);
    }
    return c;
  }
  __device__ __forceinline__ void eval4(const Row& r, const Col4& cl, int64_t, double* c) const {
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = raw(r.v, cl.v[q]) * inv;
  }
  __device__ __forceinline__ void get4(const Pre4& p, const Col4& cl, double* c) const {
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = raw(p.r.v, cl.v[q]) * inv;
  }
};

// ColorKernel with p = 2 in expanded (Gram) form, for the non-evaluation DXG sweeps:
//   a C_ij = a inv (N_i + N_j - 2 f_i.f_j),   N_j = |f_j|^2  (cost.norms)
// The row term -a inv N_i is constant along row i and cancels in the row softmax
// (dxg.py:199-202), so the sweeps evaluate
//   x'_kij = s_k (f_i.f_j) + beta_kj,  s_k = 2 a_k inv,  beta_kj = -a_k inv N_j - b_kj
// and keep the row shifts in the x' convention (shift - round(-a_k inv N_i / LSTEP)).
// Per element this is DIM FP64 for the dot product (shared by all weight sets) + 1 per
// set, instead of 2 DIM + 1 for the difference form + 1 per set.  The value the
// accessors return is the dot product f_i.f_j; beta_kj is precomputed once per sweep
// (gram_beta_kernel) and read where the difference form reads b_kj.
template <int DIM>
struct CostGram {
  static constexpr bool kStored = false;
  static constexpr bool kGram = true;
  const double* f;
  const double* nrm;
  double inv;
  int64_t n;
  struct Row { double v[DIM]; };
  struct Col { double v0[DIM], v1[DIM]; };
  // norms buffer: [|f_j - mu|^2 (n, padded to even) | centered features f_j - mu (n x DIM)]
  __device__ explicit CostGram(const CostView& v)
      : f(v.norms + ((v.n + 1) & ~int64_t(1))), nrm(v.norms), inv(v.inv_scale), n(v.n) {}
  __device__ __forceinline__ Row row(int64_t i) const {
    Row r;
#pragma unroll
    for (int d = 0; d < DIM; ++d) r.v[d] = __ldg(f + i * DIM + d);
    return r;
  }
  __device__ __forceinline__ double norm(int64_t j) const { return __ldg(nrm + j); }
  __device__ __forceinline__ Col col(int64_t j) const {
    Col c;
    int64_t j1 = j + 1 < n ? j + 1 : j;
#pragma unroll
    for (int d = 0; d < DIM; ++d) { c.v0[d] = __ldg(f + j * DIM + d); c.v1[d] = __ldg(f + j1 * DIM + d); }
    return c;
  }
  __device__ __forceinline__ static double dot(const double* a, const double* b) {
    double s = a[0] * b[0];
#pragma unroll
    for (int d = 1; d < DIM; ++d) s = fma(a[d], b[d], s);
    return s;
  }
  __device__ __forceinline__ double eval1(const Row& r, int64_t j) const {
    double b[DIM];
#pragma unroll
    for (int d = 0; d < DIM; ++d) b[d] = __ldg(f + j * DIM + d);
    return dot(r.v, b);
  }
  template <int R> struct Pre2 { Col c; };
  template <int R>
  __device__ __forceinline__ void pre2(const Row (&)[R], const Col&, int64_t j, Pre2<R>& p) const {
    col_pair<DIM>(f, j, p.c.v0, p.c.v1);
  }
  template <int R>
  __device__ __forceinline__ void get2(const Row (&rows)[R], const Col&, const Pre2<R>& p, double (&c)[R][2]) const {
#pragma unroll
    for (int r = 0; r < R; ++r) { c[r][0] = dot(rows[r].v, p.c.v0); c[r][1] = dot(rows[r].v, p.c.v1); }
  }
  struct Pre4 { Row r; };
  __device__ __forceinline__ void pre4(const Row& row, int64_t, Pre4& p) const { p.r = row; }
  struct Col4 { double v[4][DIM]; };
  __device__ __forceinline__ Col4 col4(int64_t j) const {
    Col4 c;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int64_t jj = j + q < n ? j + q : n - 1;
#pragma unroll
      for (int d = 0; d < DIM; ++d) c.v[q][d] = __ldg(f + jj * DIM + d);
    }
    return c;
  }
  __device__ __forceinline__ void eval4(const Row& r, const Col4& cl, int64_t, double* c) const {
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = dot(r.v, cl.v[q]);
  }
  __device__ __forceinline__ void get4(const Pre4& p, const Col4& cl, double* c) const {
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = dot(p.r.v, cl.v[q]);
  }
};

// GridKernel: (|drow|^P + |dcol|^P) / scale, cells row-major (core.py:200-236)
template <int P>
struct CostGrid {
  static constexpr bool kStored = false;
  static constexpr bool kGram = false;
  const double* rc;  // [row(n) | col(n)]
  double inv;
  int64_t n;
  struct Row { double r, c; };
  struct Col { double r0, c0, r1, c1; };
  __device__ explicit CostGrid(const CostView& v) : rc(v.gcoord), inv(v.inv_scale), n(v.n) {}
  __device__ __forceinline__ Row row(int64_t i) const { return Row{__ldg(rc + i), __ldg(rc + n + i)}; }
  __device__ __forceinline__ Col col(int64_t j) const {
    int64_t j1 = j + 1 < n ? j + 1 : j;
    return Col{__ldg(rc + j), __ldg(rc + n + j), __ldg(rc + j1), __ldg(rc + n + j1)};
  }
  __device__ __forceinline__ static double pw(double d) {
    d = fabs(d);
    return P == 1 ? d : (P == 2 ? d * d : d * d * d);
  }
  __device__ __forceinline__ void eval2(const Row& r, const Col& c, int64_t, double& c0, double& c1) const {
    c0 = (pw(r.r - c.r0) + pw(r.c - c.c0)) * inv;
    c1 = (pw(r.r - c.r1) + pw(r.c - c.c1)) * inv;
  }
  __device__ __forceinline__ void eval2_stream(const Row& r, const Col& c, int64_t j, double& c0, double& c1) const {
    eval2(r, c, j, c0, c1);
  }
  __device__ __forceinline__ double eval1(const Row& r, int64_t j) const {
    return (pw(r.r - __ldg(rc + j)) + pw(r.c - __ldg(rc + n + j))) * inv;
  }
  template <int R> struct Pre2 { Col c; };
  template <int R>
  __device__ __forceinline__ void pre2(const Row (&)[R], const Col&, int64_t j, Pre2<R>& p) const { p.c = col(j); }
  template <int R>
  __device__ __forceinline__ void get2(const Row (&rows)[R], const Col&, const Pre2<R>& p, double (&c)[R][2]) const {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      c[r][0] = (pw(rows[r].r - p.c.r0) + pw(rows[r].c - p.c.c0)) * inv;
      c[r][1] = (pw(rows[r].r - p.c.r1) + pw(rows[r].c - p.c.c1)) * inv;
    }
  }
  struct Pre4 { Row r; };
  __device__ __forceinline__ void pre4(const Row& row, int64_t, Pre4& p) const { p.r = row; }
  struct Col4 { double r[4], c[4]; };
  __device__ __forceinline__ Col4 col4(int64_t j) const {
    Col4 cl;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int64_t jj = j + q < n ? j + q : n - 1;
      cl.r[q] = __ldg(rc + jj);
      cl.c[q] = __ldg(rc + n + jj);
    }
    return cl;
  }
  __device__ __forceinline__ void eval4(const Row& r, const Col4& cl, int64_t, double* c) const {
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = (pw(r.r - cl.r[q]) + pw(r.c - cl.c[q])) * inv;
  }
  __device__ __forceinline__ void get4(const Pre4& p, const Col4& cl, double* c) const {
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = (pw(p.r.r - cl.r[q]) + pw(p.r.c - cl.c[q])) * inv;
  }
};

// Dispatch a functor templated on the provider type for a runtime cost descriptor.
// F::template run<COST>() must be callable; returns false for unsupported combos.
#define LEANOT_DISPATCH_COST(view, FN)                                        \
  [&]() -> int {                                                               \
    switch ((view).kind) {                                                     \
      case LEANOT_COST_STORED: return FN.template run<CostStored>();           \
      case LEANOT_COST_GRID:                                                   \
        if ((view).p == 1) return FN.template run<CostGrid<1>>();              \
        if ((view).p == 2) return FN.template run<CostGrid<2>>();              \
        if ((view).p == 3) return FN.template run<CostGrid<3>>();              \
        return LEANOT_EINVAL;                                                  \
      case LEANOT_COST_POINTS:                                                 \
        if ((view).dim == 1 && (view).p == 1) return FN.template run<CostPoints<1, 1>>(); \
        if ((view).dim == 1 && (view).p == 2) return FN.template run<CostPoints<1, 2>>(); \
        if ((view).dim == 1 && (view).p == 3) return FN.template run<CostPoints<1, 3>>(); \
        if ((view).dim == 2 && (view).p == 1) return FN.template run<CostPoints<2, 1>>(); \
        if ((view).dim == 2 && (view).p == 2) return FN.template run<CostPoints<2, 2>>(); \
        if ((view).dim == 2 && (view).p == 3) return FN.template run<CostPoints<2, 3>>(); \
        if ((view).dim == 3 && (view).p == 1) return FN.template run<CostPoints<3, 1>>(); \
        if ((view).dim == 3 && (view).p == 2) return FN.template run<CostPoints<3, 2>>(); \
        if ((view).dim == 3 && (view).p == 3) return FN.template run<CostPoints<3, 3>>(); \
        if ((view).dim == 4 && (view).p == 1) return FN.template run<CostPoints<4, 1>>(); \
        if ((view).dim == 4 && (view).p == 2) return FN.template run<CostPoints<4, 2>>(); \
        if ((view).dim == 4 && (view).p == 3) return FN.template run<CostPoints<4, 3>>(); \
        return LEANOT_EINVAL;                                                  \
      default: return LEANOT_EINVAL;                                           \
    }                                                                          \
  }()

}  // namespace leanot
