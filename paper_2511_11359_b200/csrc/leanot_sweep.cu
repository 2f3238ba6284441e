// n^2 sweeps of the DXG hot path on sm_100a (two-pass form).
//
//  pass A (rowpass_kernel): per row i and weight set k
//      S_ki = sum_j exp(x_kij - m_ki*LSTEP),  x_kij = -(a_k C_ij + b_kj)
//    with the integer shift m_ki taken from the previous iteration's row
//    log-normalizer (SURVEY.md §7 hard part 4), so no row-max pass is needed.
//    Evaluation sweeps also accumulate sum e*C, sum e*x (-> _plan_stats,
//    dxg.py:282-310) and min_j (C_ij + sd_j) (-> dual_penalized_value at eta=0,
//    dxg.py:344-348) for weight set 0.
//  pass B (colpass_kernel): col_kj = sum_i (r_i/S_ki) exp(x_kij - m_ki*LSTEP)
//    (column_marginal, dxg.py:193-208) for all K weight sets from one read of
//    each C element; each CTA owns a 512-column tile and a row split and writes a
//    partial slab; slabs are reduced in fixed order (deterministic, no atomics).
//
// Both weight sets of a DXG iteration (current and midpoint weights) are swept
// together: the midpoint weights depend only on the current state (dxg.py:274).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "leanot_cost.cuh"
#include "leanot_internal.h"

namespace leanot {

#ifndef LEANOT_RP_R
#define LEANOT_RP_R 4     // rows per pass-A CTA step (K <= 2)
#endif
#ifndef LEANOT_RP_MINB
#define LEANOT_RP_MINB 2  // pass-A CTAs per SM the register budget targets
#endif
#ifndef LEANOT_CP_SROW
#define LEANOT_CP_SROW 1  // pass B, on-the-fly costs: row data staged in shared memory per chunk
#endif
#ifndef LEANOT_CP_MINB
#define LEANOT_CP_MINB 2  // pass-B CTAs per SM the register budget targets
#endif
constexpr int RP_THREADS = 256;
constexpr int CP_THREADS = 256;
constexpr int CP_V = 4;                  // columns per thread in the column pass
constexpr int CP_TILE = CP_V * CP_THREADS;  // columns per column-pass tile
constexpr int CP_CHUNK = 128;            // rows staged per smem chunk

// S outside [2^-900, 2^900] (or NaN) means the shift was far from the row's
// log-normalizer: the row is recomputed with an exact max shift (fixup_kernel).
__device__ __forceinline__ bool sum_ok(double S) { return S >= 0x1p-900 && S <= 0x1p900; }

// Integer part (units of LSTEP) of the row term -a_k inv N_i that the expanded form
// drops (CostGram); identical expression wherever it is evaluated.
__device__ __forceinline__ int64_t gram_off(double a_k, double inv, double N_i) {
  return llrint(((-a_k) * inv) * N_i * (1.0 / LSTEP));
}

// m: the row shift in the x convention (shift_next derives from it); mu: the shift the
// sweep actually used, stored for pass B (mu = m except for the expanded form).
__device__ __forceinline__ void finalize_row(const RowPassArgs& A, int k, int64_t li, double S, int64_t m,
                                             int64_t mu) {
  const int64_t nr = A.i1 - A.i0;
  A.S[k * nr + li] = S;
  if (A.m_used) A.m_used[k * nr + li] = mu;
  if (!sum_ok(S)) {
    int slot = atomicAdd(A.flags, 1);
    A.flags[2 + 2 * slot] = k;
    A.flags[3 + 2 * slot] = (int)li;
    return;
  }
  if (A.coef) {
    double g = A.rw ? A.rw[A.i0 + li] / S : 1.0 / S;
    double* cf = A.coef + (k * nr + li) * 4;
    cf[0] = g * EC0; cf[1] = g * EC1; cf[2] = g * EC2; cf[3] = g * EC3;
  }
  if (A.shift_next && (A.next_group > 0 ? k % A.next_group == A.next_from_k : k == A.next_from_k))
    A.shift_next[(A.next_group > 0 ? (int64_t)(k / A.next_group) * nr : 0) + li] = m + llrint(log(S) * (1.0 / LSTEP));
}

template <class COST, int K, int R, bool EVAL>
__global__ void __launch_bounds__(RP_THREADS, LEANOT_RP_MINB) rowpass_kernel(const RowPassArgs A, int64_t rb0, int64_t rb1) {
  // this launch finalizes rows [rb0, rb1) of [A.i0, A.i1) (local indices stay relative to A.i0)
  extern __shared__ __align__(16) char smem[];
  constexpr int NV = R * K + (EVAL ? 3 * R : 0);
  __shared__ double red[RP_THREADS / 32][NV];
  load_table(reinterpret_cast<double*>(smem));
  __syncthreads();
  const uint32_t tb = lane_tab_addr(smem);
  const COST cost(A.cost);
  const int64_t n = A.cost.n;
  const int64_t nr = A.i1 - A.i0;
  const int64_t nblk = (rb1 - rb0 + R - 1) / R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  static_assert(!(EVAL && COST::kGram), "evaluation sweeps need C itself");
  // x = mult_k * c + nb_kj: c = C_ij, mult = -a_k, nb = -b_kj; expanded form (CostGram):
  // c = f_i.f_j, mult = 2 a_k inv, nb = beta_kj (A.b[k] points at beta_k)
  double mult[K];
#pragma unroll
  for (int k = 0; k < K; ++k) mult[k] = COST::kGram ? 2.0 * A.a[k] * A.cost.inv_scale : -A.a[k];

  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t ib = rb0 + blk * R;
    typename COST::Row rows[R];
    uint32_t mlo[R][K];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      int64_t i = ib + r < rb1 ? ib + r : rb1 - 1;
      rows[r] = cost.row(i);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        int64_t sh = shift_at(A, k, i - A.i0);
        if constexpr (COST::kGram) sh -= gram_off(A.a[k], A.cost.inv_scale, cost.norm(i));
        mlo[r][k] = (uint32_t)sh;
      }
    }
    double acc[R][K];
    double U[R], V[R], mn[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      U[r] = 0.0; V[r] = 0.0; mn[r] = INFINITY;
#pragma unroll
      for (int k = 0; k < K; ++k) acc[r][k] = 0.0;
    }
    const int64_t nev = n & ~int64_t(1);
    // Software pipeline, ping-pong: the loads of step s+1 are in flight while step s
    // computes; two named buffers (no register copies between iterations).
    const typename COST::Col cl0{};
    typename COST::template Pre2<R> pa, pb;
    double2 ba[K], bb[K], sda = make_double2(0.0, 0.0), sdb = make_double2(0.0, 0.0);
    const int64_t stride = 2 * RP_THREADS;
    int64_t j = 2 * threadIdx.x;
    auto fetch = [&](int64_t jj, typename COST::template Pre2<R>& p, double2 (&bv)[K], double2& sdv) {
      cost.pre2(rows, cl0, jj, p);
#pragma unroll
      for (int k = 0; k < K; ++k) bv[k] = __ldg(reinterpret_cast<const double2*>(A.b[k] + jj));
      if (EVAL) sdv = __ldg(reinterpret_cast<const double2*>(A.sd + jj));
    };
    auto compute = [&](const typename COST::template Pre2<R>& p, const double2 (&bv)[K], const double2& sdv) {
      double cc[R][2];
      cost.get2(rows, cl0, p, cc);
      double2 nbv[K];
#pragma unroll
      for (int k = 0; k < K; ++k) nbv[k] = COST::kGram ? bv[k] : make_double2(-bv[k].x, -bv[k].y);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double c0 = cc[r][0], c1 = cc[r][1];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const double x0 = fma(mult[k], c0, nbv[k].x);
          const double x1 = fma(mult[k], c1, nbv[k].y);
          if (EVAL && k == 0) {
            const double e0 = texp(tb, x0, mlo[r][0]);
            const double e1 = texp(tb, x1, mlo[r][0]);
            acc[r][0] += e0 + e1;
            U[r] = fma(e0, c0, fma(e1, c1, U[r]));
            V[r] = fma(e0, x0, fma(e1, x1, V[r]));
            mn[r] = fmin(mn[r], fmin(c0 + sdv.x, c1 + sdv.y));
          } else {
            texp_acc(tb, x0, mlo[r][k], acc[r][k]);
            texp_acc(tb, x1, mlo[r][k], acc[r][k]);
          }
        }
      }
    };
    if (j < nev) fetch(j, pa, ba, sda);
    // steady state: two steps per trip
    for (; j + stride < nev; j += 2 * stride) {
      fetch(j + stride, pb, bb, sdb);
      compute(pa, ba, sda);
      if (j + 2 * stride < nev) fetch(j + 2 * stride, pa, ba, sda);
      compute(pb, bb, sdb);
    }
    if (j < nev) compute(pa, ba, sda);
    if ((n & 1) && threadIdx.x == 0) {  // odd tail column
      const int64_t j = n - 1;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double c0 = cost.eval1(rows[r], j);
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const double bj = __ldg(A.b[k] + j);
          double x0 = fma(mult[k], c0, COST::kGram ? bj : -bj);
          double e0 = texp(tb, x0, mlo[r][k]);
          acc[r][k] += e0;
          if (EVAL && k == 0) {
            U[r] = fma(e0, c0, U[r]);
            V[r] = fma(e0, x0, V[r]);
            mn[r] = fmin(mn[r], c0 + __ldg(A.sd + j));
          }
        }
      }
    }
    // block reduction in fixed order (deterministic)
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double v = warp_sum(acc[r][k]);
        if (lane == 0) red[warp][r * K + k] = v;
      }
      if (EVAL) {
        double u = warp_sum(U[r]), vv = warp_sum(V[r]), m = warp_min(mn[r]);
        if (lane == 0) {
          red[warp][R * K + 3 * r] = u;
          red[warp][R * K + 3 * r + 1] = vv;
          red[warp][R * K + 3 * r + 2] = m;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x < NV) {
      const int v = threadIdx.x;
      const bool is_min = EVAL && v >= R * K && ((v - R * K) % 3 == 2);
      double t = red[0][v];
      for (int w = 1; w < RP_THREADS / 32; ++w) t = is_min ? fmin(t, red[w][v]) : t + red[w][v];
      if (v < R * K) {
        const int r = v / K, k = v % K;
        const int64_t i = ib + r;
        if (i < rb1) {
          const int64_t m = shift_at(A, k, i - A.i0);
          int64_t mu = m;
          if constexpr (COST::kGram) mu -= gram_off(A.a[k], A.cost.inv_scale, cost.norm(i));
          finalize_row(A, k, i - A.i0, t, m, mu);
        }
      } else if (EVAL) {
        const int q = v - R * K, r = q / 3, s = q % 3;
        const int64_t i = ib + r;
        if (i < rb1) A.rowstat[s * nr + (i - A.i0)] = t;
      }
    }
    __syncthreads();
  }
}

// Exact recompute of rows whose shifted sum left the safe range (rare: first
// sweeps of injected states, pathological step sizes).  One CTA, loops the list.
template <class COST>
__global__ void __launch_bounds__(1024) fixup_kernel(const RowPassArgs A) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double red[32];
  __shared__ double red3[32][2];
  __shared__ double bcast;
  const int cnt = *A.flags;
  if (cnt == 0) return;
  load_table(reinterpret_cast<double*>(smem));
  __syncthreads();
  const uint32_t tb = lane_tab_addr(smem);
  const COST cost(A.cost);
  const int64_t n = A.cost.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = 0; e < cnt; ++e) {
    const int k = A.flags[2 + 2 * e];
    const int64_t li = A.flags[3 + 2 * e];
    const int64_t i = A.i0 + li;
    const typename COST::Row row = cost.row(i);
    const double mult = COST::kGram ? 2.0 * A.a[k] * A.cost.inv_scale : -A.a[k];
    auto xval = [&](int64_t j) { return fma(mult, cost.eval1(row, j), COST::kGram ? A.b[k][j] : -A.b[k][j]); };
    double mx = -INFINITY;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) mx = fmax(mx, xval(j));
    mx = warp_max(mx);
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red[0];
      for (int w = 1; w < nw; ++w) t = fmax(t, red[w]);
      bcast = t;
    }
    __syncthreads();
    const int64_t m = llrint(bcast * (1.0 / LSTEP));
    const uint32_t mlo = (uint32_t)m;
    // evaluation sweeps: the row's plan statistics (sum e*C, sum e*x; dxg.py:282-310) were
    // accumulated by pass A with the rejected shift, so they are recomputed with this one
    const bool stats = !COST::kGram && A.rowstat && k == 0;
    double s = 0.0, u = 0.0, v = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      const double c = cost.eval1(row, j);
      const double x = fma(mult, c, COST::kGram ? A.b[k][j] : -A.b[k][j]);
      const double e = texp(tb, x, mlo);
      s += e;
      if (stats) { u = fma(e, c, u); v = fma(e, x, v); }
    }
    s = warp_sum(s);
    if (stats) { u = warp_sum(u); v = warp_sum(v); }
    __syncthreads();
    if (lane == 0) { red[warp] = s; red3[warp][0] = u; red3[warp][1] = v; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red[0];
      for (int w = 1; w < nw; ++w) t += red[w];
      if (stats) {
        const int64_t nr = A.i1 - A.i0;
        double tu = red3[0][0], tv = red3[0][1];
        for (int w = 1; w < nw; ++w) { tu += red3[w][0]; tv += red3[w][1]; }
        A.rowstat[li] = tu;
        A.rowstat[nr + li] = tv;
      }
      // finalize without re-flagging
      const int64_t nr = A.i1 - A.i0;
      A.S[k * nr + li] = t;
      if (A.m_used) A.m_used[k * nr + li] = m;
      if (A.coef) {
        double g = A.rw ? A.rw[i] / t : 1.0 / t;
        double* cf = A.coef + (k * nr + li) * 4;
        cf[0] = g * EC0; cf[1] = g * EC1; cf[2] = g * EC2; cf[3] = g * EC3;
      }
      // expanded form: m is in the x' convention; the stored shift is in the x convention
      int64_t off = 0;
      if constexpr (COST::kGram) off = gram_off(A.a[k], A.cost.inv_scale, cost.norm(i));
      if (A.shift_next && (A.next_group > 0 ? k % A.next_group == A.next_from_k : k == A.next_from_k))
        A.shift_next[(A.next_group > 0 ? (int64_t)(k / A.next_group) * nr : 0) + li] =
            m + off + llrint(log(t) * (1.0 / LSTEP));
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *A.flags = 0;
}

// Row maxima of x_kij -> integer shifts (robust start for injected states).
template <class COST, int K>
__global__ void __launch_bounds__(RP_THREADS) rowmax_kernel(const RowPassArgs A, int64_t* shift_out) {
  __shared__ double red[RP_THREADS / 32][K];
  const COST cost(A.cost);
  const int64_t n = A.cost.n, nr = A.i1 - A.i0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double na[K];
#pragma unroll
  for (int k = 0; k < K; ++k) na[k] = -A.a[k];
  for (int64_t i = A.i0 + blockIdx.x; i < A.i1; i += gridDim.x) {
    const typename COST::Row row = cost.row(i);
    double mx[K];
#pragma unroll
    for (int k = 0; k < K; ++k) mx[k] = -INFINITY;
    for (int64_t j = threadIdx.x; j < n; j += RP_THREADS) {
      double c = cost.eval1(row, j);
#pragma unroll
      for (int k = 0; k < K; ++k) mx[k] = fmax(mx[k], fma(na[k], c, -__ldg(A.b[k] + j)));
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double v = warp_max(mx[k]);
      if (lane == 0) red[warp][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < K) {
      double t = red[0][threadIdx.x];
      for (int w = 1; w < RP_THREADS / 32; ++w) t = fmax(t, red[w][threadIdx.x]);
      shift_out[threadIdx.x * nr + (i - A.i0)] = llrint(t * (1.0 / LSTEP));
    }
    __syncthreads();
  }
}

// pass B: column sums for K weight sets over a row split, written to a slab.
// Each thread owns 4 consecutive columns (two 16-byte loads per row for the stored
// cost); per-row constants (shift, g*EC0..3) are staged in shared memory and read
// as broadcasts.
template <class COST, int K>
__global__ void __launch_bounds__(CP_THREADS, LEANOT_CP_MINB) colpass_kernel(const ColPassArgs A) {
  extern __shared__ __align__(16) char smem[];
  double* s_coef = reinterpret_cast<double*>(smem + TAB_BYTES);            // [CP_CHUNK][K][4]
  uint32_t* s_m = reinterpret_cast<uint32_t*>(s_coef + CP_CHUNK * K * 4);  // [CP_CHUNK][K]
  // on-the-fly costs: the chunk's row data (features / grid coordinates) staged with the
  // row constants, so the inner loop reads it as shared-memory broadcasts
  typename COST::Row* s_row = reinterpret_cast<typename COST::Row*>(s_m + CP_CHUNK * K);  // [CP_CHUNK]
  load_table(reinterpret_cast<double*>(smem));
  __syncthreads();
  const uint32_t tb = lane_tab_addr(smem);
  const COST cost(A.cost);
  const int64_t n = A.cost.n, nr = A.i1 - A.i0;
  const int64_t ntiles = (n + CP_TILE - 1) / CP_TILE;
  const int64_t items = ntiles * A.splits;
  const int64_t rows_per_split = (nr + A.splits - 1) / A.splits;
  double mult[K];
#pragma unroll
  for (int k = 0; k < K; ++k) mult[k] = COST::kGram ? 2.0 * A.a[k] * A.cost.inv_scale : -A.a[k];

  // columns of this thread: CP_V consecutive ones
  auto colv = [&](int64_t tile, int v) -> int64_t { return tile * CP_TILE + CP_V * threadIdx.x + v; };
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t tile = it % ntiles, split = it / ntiles;
    const int64_t j = colv(tile, 0);
    // columns are increasing in v: the thread's valid columns are v < nv
    int nv = 0;
#pragma unroll
    for (int v = 0; v < CP_V; ++v) nv += colv(tile, v) < n ? 1 : 0;
    const bool full = nv == CP_V;
    const int64_t jl = nv > 0 ? j : 0;
    const typename COST::Col4 cl = cost.col4(jl);
    double nb[K][CP_V];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int v = 0; v < CP_V; ++v)
        nb[k][v] = v < nv ? (COST::kGram ? 1.0 : -1.0) * __ldg(A.b[k] + colv(tile, v)) : 0.0;
    double acc[K][CP_V];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int v = 0; v < CP_V; ++v) acc[k][v] = 0.0;
    const int64_t rs0 = A.i0 + split * rows_per_split;
    const int64_t rs1 = A.i1 < rs0 + rows_per_split ? A.i1 : rs0 + rows_per_split;
    for (int64_t q0 = rs0; q0 < rs1; q0 += CP_CHUNK) {
      const int nq = (int)(rs1 - q0 < CP_CHUNK ? rs1 - q0 : CP_CHUNK);
      __syncthreads();
      for (int t = threadIdx.x; t < nq * K * 4; t += CP_THREADS) {
        int q = t / (K * 4), k = (t / 4) % K, c = t % 4;
        s_coef[t] = A.coef[(k * nr + (q0 - A.i0 + q)) * 4 + c];
      }
      for (int t = threadIdx.x; t < nq * K; t += CP_THREADS) {
        int q = t / K, k = t % K;
        s_m[t] = (uint32_t)A.m[k * nr + (q0 - A.i0 + q)];
      }
      if constexpr (!COST::kStored && LEANOT_CP_SROW)
        for (int t = threadIdx.x; t < nq; t += CP_THREADS) s_row[t] = cost.row(q0 + t);
      __syncthreads();
      if (full) {
        // 2-row ping-pong: rows (q, q+1) compute while rows (q+2, q+3) load
        typename COST::Row row = cost.row(q0);
        typename COST::Pre4 pa0, pa1, pb0, pb1;
        auto fetch = [&](typename COST::Pre4& p, int q) {
          if (q < nq) {
            if constexpr (COST::kStored) cost.pre4(row, j, p);
            else if constexpr (LEANOT_CP_SROW) cost.pre4(s_row[q], j, p);
            else cost.pre4(cost.row(q0 + q), j, p);
          }
          if constexpr (COST::kStored) row.p += cost.ld;
        };
        auto compute = [&](const typename COST::Pre4& p, int q) {
          double c[CP_V];
          cost.get4(p, cl, c);
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const double2 g01 = *reinterpret_cast<const double2*>(s_coef + (q * K + k) * 4);
            const double2 g23 = *reinterpret_cast<const double2*>(s_coef + (q * K + k) * 4 + 2);
            const uint32_t mlo = s_m[q * K + k];
#pragma unroll
            for (int v = 0; v < CP_V; ++v)
              texp_gacc(tb, fma(mult[k], c[v], nb[k][v]), mlo, g01.x, g01.y, g23.x, g23.y, acc[k][v]);
          }
        };
        fetch(pa0, 0);
        fetch(pa1, 1);
        int q = 0;
        for (; q + 2 < nq; q += 4) {
          fetch(pb0, q + 2);
          fetch(pb1, q + 3);
          compute(pa0, q);
          compute(pa1, q + 1);
          fetch(pa0, q + 4);
          fetch(pa1, q + 5);
          compute(pb0, q + 2);
          if (q + 3 < nq) compute(pb1, q + 3);
        }
        if (q < nq) compute(pa0, q);
        if (q + 1 < nq) compute(pa1, q + 1);
      } else if (nv > 0) {
        for (int q = 0; q < nq; ++q) {
          const typename COST::Row row = cost.row(q0 + q);
#pragma unroll
          for (int v = 0; v < CP_V; ++v) {
            if (v < nv) {
              const double cv = cost.eval1(row, colv(tile, v));
#pragma unroll
              for (int k = 0; k < K; ++k) {
                const double* cf = s_coef + (q * K + k) * 4;
                texp_gacc(tb, fma(mult[k], cv, nb[k][v]), s_m[q * K + k], cf[0], cf[1], cf[2], cf[3],
                          acc[k][v]);
              }
            }
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double* out = A.slab + (split * K + k) * n;
#pragma unroll
      for (int v = 0; v < CP_V; ++v)
        if (v < nv) out[colv(tile, v)] = acc[k][v];
    }
  }
}

// col[k][j] = sum over splits in a fixed order: 32 outputs x 8 split groups per block; group g
// adds splits g, g+8, ... in increasing order, then the 8 group sums are added in group order.
__global__ void __launch_bounds__(256) slab_reduce_kernel(const double* __restrict__ slab, int splits, int K,
                                                          int64_t n, double* __restrict__ col) {
  __shared__ double part[8][33];
  const int64_t total = (int64_t)K * n;
  const int o = threadIdx.x & 31, g = threadIdx.x >> 5;
  for (int64_t t0 = (int64_t)blockIdx.x * 32; t0 < total; t0 += (int64_t)gridDim.x * 32) {
    const int64_t t = t0 + o;
    double s = 0.0;
    if (t < total)
      for (int q = g; q < splits; q += 8) s += slab[q * total + t];
    part[g][o] = s;
    __syncthreads();
    if (g == 0 && t < total) {
      double v = part[0][o];
#pragma unroll
      for (int h = 1; h < 8; ++h) v += part[h][o];
      col[t] = v;
    }
    __syncthreads();
  }
}

// Row LSE with exact max, for the entropic dual / potentials / barycenter dual:
//   L_i = LSE_j( (sgn * C_ij + v_j) * scale )   (dxg.py:337, 367; barycenter.py:189)
// two reads of the row (max, then shifted sum); evaluation-only.
template <class COST>
__global__ void __launch_bounds__(RP_THREADS) rowlse_kernel(const CostView cv, int64_t i0, int64_t i1, const double* v,
                                                           double sgn, double scale, const double* vmin, double* L) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double red[RP_THREADS / 32];
  __shared__ double bc;
  load_table(reinterpret_cast<double*>(smem));
  __syncthreads();
  const uint32_t tb = lane_tab_addr(smem);
  const COST cost(cv);
  const int64_t n = cv.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t i = i0 + blockIdx.x; i < i1; i += gridDim.x) {
    const typename COST::Row row = cost.row(i);
    double xm;
    if (vmin) {
      // max_j fl(x_j * scale) = fl(min_j x_j * scale) for scale < 0 (rounding is monotone),
      // so pass A's row minimum gives the exact max without a first read of the row
      xm = vmin[i - i0] * scale;
    } else {
      double mx = -INFINITY;
      for (int64_t j = threadIdx.x; j < n; j += RP_THREADS) mx = fmax(mx, (sgn * cost.eval1(row, j) + __ldg(v + j)) * scale);
      mx = warp_max(mx);
      if (lane == 0) red[warp] = mx;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = red[0];
        for (int w = 1; w < RP_THREADS / 32; ++w) t = fmax(t, red[w]);
        bc = t;
      }
      __syncthreads();
      xm = bc;
    }
    double s = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += RP_THREADS) {
      double y = (sgn * cost.eval1(row, j) + __ldg(v + j)) * scale - xm;
      texp_acc(tb, fmin(fmax(y, -1000.0), 0.0), 0u, s);  // y <= 0 whenever xm is the exact max
    }
    s = warp_sum(s);
    __syncthreads();
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red[0];
      for (int w = 1; w < RP_THREADS / 32; ++w) t += red[w];
      L[i - i0] = xm + log(t);
    }
    __syncthreads();
  }
}

// min_j (C_ij + v_j) per row (dxg.py:344-348)
template <class COST>
__global__ void __launch_bounds__(RP_THREADS) rowmin_kernel(const CostView cv, int64_t i0, int64_t i1, const double* v, double* out) {
  __shared__ double red[RP_THREADS / 32];
  const COST cost(cv);
  const int64_t n = cv.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t i = i0 + blockIdx.x; i < i1; i += gridDim.x) {
    const typename COST::Row row = cost.row(i);
    double mn = INFINITY;
    for (int64_t j = threadIdx.x; j < n; j += RP_THREADS) mn = fmin(mn, cost.eval1(row, j) + __ldg(v + j));
    mn = warp_min(mn);
    if (lane == 0) red[warp] = mn;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red[0];
      for (int w = 1; w < RP_THREADS / 32; ++w) t = fmin(t, red[w]);
      out[i - i0] = t;
    }
    __syncthreads();
  }
}

// CostKernel.block: rows [i0,i1) of the normalized cost
template <class COST>
__global__ void cost_block_kernel(const CostView cv, int64_t i0, int64_t i1, double* out, int64_t ldo) {
  const COST cost(cv);
  const int64_t n = cv.n;
  for (int64_t i = i0 + blockIdx.y; i < i1; i += gridDim.y) {
    const typename COST::Row row = cost.row(i);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
      out[(i - i0) * ldo + j] = cost.eval1(row, j);
  }
}

// LEANOT_TMA=0 disables the TMA-staged stored-cost kernels (A/B comparisons)
static bool tma_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LEANOT_TMA");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// LEANOT_GRAM=0 keeps the difference form for squared-Euclidean point costs (A/B comparisons)
bool gram_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LEANOT_GRAM");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static bool tma_cols_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LEANOT_TMA_COLS");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

int num_sms();

}  // namespace leanot

#include "leanot_sweep_tma.cu"

namespace leanot {

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------

int g_num_sms = 0;

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

// LEANOT_RP_TAIL=0 disables the pass-A wave-tail split (A/B measurements)
static bool tail_split_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LEANOT_RP_TAIL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <class COST, int K, int R, bool EVAL>
static int launch_rowpass_t(const RowPassArgs& A, cudaStream_t st) {
  auto kern = rowpass_kernel<COST, K, R, EVAL>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TAB_BYTES) != cudaSuccess) return LEANOT_ECUDA;
    attr = true;
  }
  static int occ = 0;
  if (occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, RP_THREADS, TAB_BYTES) != cudaSuccess || occ < 1) occ = 1;
  }
  const int64_t nr = A.i1 - A.i0;
  const int64_t nblk = (nr + R - 1) / R;
  const int64_t slots = (int64_t)num_sms() * occ;
  int grid = (int)std::min<int64_t>(nblk, slots);
  if (grid < 1) return LEANOT_OK;
  // Wave tail: when the last wave of R-row blocks would fill at most half the slots, the
  // remaining rows run as a second launch of R/2-row blocks (one wave of half-length
  // blocks instead of a half-empty full-length one).  Row sums do not depend on R (same
  // per-thread column order, same reductions), so the split is bitwise neutral.
  if constexpr (R % 2 == 0) {
    const int64_t full = (nblk / slots) * slots, rem = nblk - full;
    if (full > 0 && rem > 0 && 2 * rem <= slots && tail_split_enabled()) {
      const int64_t rmid = A.i0 + full * R;
      kern<<<grid, RP_THREADS, TAB_BYTES, st>>>(A, A.i0, rmid);
      auto kern2 = rowpass_kernel<COST, K, R / 2, EVAL>;
      static bool attr2 = false;
      if (!attr2) {
        if (cudaFuncSetAttribute(kern2, cudaFuncAttributeMaxDynamicSharedMemorySize, TAB_BYTES) != cudaSuccess)
          return LEANOT_ECUDA;
        attr2 = true;
      }
      const int64_t nb2 = (A.i1 - rmid + R / 2 - 1) / (R / 2);
      kern2<<<(int)std::min<int64_t>(nb2, slots), RP_THREADS, TAB_BYTES, st>>>(A, rmid, A.i1);
      return LEANOT_OK;
    }
  }
  kern<<<grid, RP_THREADS, TAB_BYTES, st>>>(A, A.i0, A.i1);
  return LEANOT_OK;
}

template <class COST>
static int launch_fixup_t(const RowPassArgs& A, cudaStream_t st) {
  auto kern = fixup_kernel<COST>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TAB_BYTES) != cudaSuccess) return LEANOT_ECUDA;
    attr = true;
  }
  kern<<<1, 1024, TAB_BYTES, st>>>(A);
  return LEANOT_OK;
}

// squared-Euclidean point costs -> their expanded-form provider (CostGram)
template <class C> struct GramOf { using type = void; };
template <int D> struct GramOf<CostPoints<D, 2>> { using type = CostGram<D>; };

struct RowPassFn {
  const RowPassArgs& A;
  int K;
  bool eval;
  cudaStream_t st;
  template <class COST>
  int run() {
    int rc;
    constexpr int R = LEANOT_RP_R;
    using G = typename GramOf<COST>::type;
    if constexpr (!std::is_void<G>::value) {
      if (!eval && A.gram && A.cost.norms) {
        if (K == 1) rc = launch_rowpass_t<G, 1, R, false>(A, st);
        else if (K == 2) rc = launch_rowpass_t<G, 2, R, false>(A, st);
        else return LEANOT_EINVAL;
        if (rc != LEANOT_OK) return rc;
        if (A.flags) return launch_fixup_t<G>(A, st);
        return LEANOT_OK;
      }
    }
    if constexpr (std::is_same<COST, CostStored>::value) {
      if (tma_ok(A.cost) && (K == 1 || K == 2 || (K == 4 && !eval))) {
        if (K == 1) rc = eval ? launch_rowpass_tma_t<1, 4, true>(A, st) : launch_rowpass_tma_t<1, 4, false>(A, st);
        else if (K == 2) rc = eval ? launch_rowpass_tma_t<2, 4, true>(A, st) : launch_rowpass_tma_t<2, 4, false>(A, st);
        else rc = launch_rowpass_tma_t<4, 2, false>(A, st);   // two barycenter marginals per read of C
        if (rc != LEANOT_OK) return rc;
        if (A.flags) return launch_fixup_t<COST>(A, st);
        return LEANOT_OK;
      }
    }
    if (K == 1) rc = eval ? launch_rowpass_t<COST, 1, R, true>(A, st) : launch_rowpass_t<COST, 1, R, false>(A, st);
    else if (K == 2) rc = eval ? launch_rowpass_t<COST, 2, R, true>(A, st) : launch_rowpass_t<COST, 2, R, false>(A, st);
    else if (K == 4 && !eval) rc = launch_rowpass_t<COST, 4, 2, false>(A, st);
    else return LEANOT_EINVAL;
    if (rc != LEANOT_OK) return rc;
    if (A.flags) return launch_fixup_t<COST>(A, st);
    return LEANOT_OK;
  }
};

int launch_rowpass(const RowPassArgs& A, int K, bool eval, cudaStream_t st) {
  RowPassFn f{A, K, eval, st};
  return LEANOT_DISPATCH_COST(A.cost, f);
}

struct RowMaxFn {
  const RowPassArgs& A;
  int K;
  int64_t* out;
  cudaStream_t st;
  template <class COST>
  int run() {
    const int64_t nr = A.i1 - A.i0;
    int grid = (int)std::min<int64_t>(nr, (int64_t)num_sms() * 8);
    if (grid < 1) return LEANOT_OK;
    if (K == 1) rowmax_kernel<COST, 1><<<grid, RP_THREADS, 0, st>>>(A, out);
    else if (K == 2) rowmax_kernel<COST, 2><<<grid, RP_THREADS, 0, st>>>(A, out);
    else return LEANOT_EINVAL;
    return LEANOT_OK;
  }
};

int launch_rowmax(const RowPassArgs& A, int K, int64_t* out, cudaStream_t st) {
  RowMaxFn f{A, K, out, st};
  return LEANOT_DISPATCH_COST(A.cost, f);
}

template <class COST, int K>
static int launch_colpass_t(const ColPassArgs& A, cudaStream_t st) {
  auto kern = colpass_kernel<COST, K>;
  const int smem = TAB_BYTES + CP_CHUNK * K * 4 * 8 + CP_CHUNK * K * 4 + (int)(CP_CHUNK * sizeof(typename COST::Row));
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return LEANOT_ECUDA;
    attr = true;
  }
  static int occ = 0;
  if (occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, CP_THREADS, smem) != cudaSuccess || occ < 1) occ = 1;
  }
  const int64_t n = A.cost.n;
  const int64_t items = ((n + CP_TILE - 1) / CP_TILE) * A.splits;
  int grid = (int)std::min<int64_t>(items, (int64_t)num_sms() * occ);
  if (grid < 1) return LEANOT_OK;
  kern<<<grid, CP_THREADS, smem, st>>>(A);
  return LEANOT_OK;
}

struct ColPassFn {
  const ColPassArgs& A;
  int K;
  cudaStream_t st;
  template <class COST>
  int run() {
    using G = typename GramOf<COST>::type;
    if constexpr (!std::is_void<G>::value) {
      if (A.gram && A.cost.norms) {
        if (K == 1) return launch_colpass_t<G, 1>(A, st);
        if (K == 2) return launch_colpass_t<G, 2>(A, st);
        return LEANOT_EINVAL;
      }
    }
    if constexpr (std::is_same<COST, CostStored>::value) {
      // the TMA column pass is kept for experiments (LEANOT_TMA_COLS=1); measured slower
      // than the register-pipelined one (profiles/r01_tma.md)
      if (tma_ok(A.cost) && tma_cols_enabled()) {
        if (K == 1) return launch_colpass_tma_t<1>(A, st);
        if (K == 2) return launch_colpass_tma_t<2>(A, st);
      }
    }
    if (K == 1) return launch_colpass_t<COST, 1>(A, st);
    if (K == 2) return launch_colpass_t<COST, 2>(A, st);
    if (K == 4) return launch_colpass_t<COST, 4>(A, st);
    return LEANOT_EINVAL;
  }
};

int launch_colpass(const ColPassArgs& A, int K, cudaStream_t st) {
  ColPassFn f{A, K, st};
  return LEANOT_DISPATCH_COST(A.cost, f);
}

int launch_slab_reduce(const double* slab, int splits, int K, int64_t n, double* col, cudaStream_t st) {
  const int64_t total = (int64_t)K * n;
  int grid = (int)std::min<int64_t>((total + 31) / 32, (int64_t)num_sms() * 8);
  if (grid < 1) return LEANOT_OK;
  slab_reduce_kernel<<<grid, 256, 0, st>>>(slab, splits, K, n, col);
  return LEANOT_OK;
}

struct RowLseFn {
  const CostView& cv;
  int64_t i0, i1;
  const double* v;
  double sgn, scale;
  const double* vmin;
  double* L;
  cudaStream_t st;
  template <class COST>
  int run() {
    auto kern = rowlse_kernel<COST>;
    static bool attr = false;
    if (!attr) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TAB_BYTES) != cudaSuccess) return LEANOT_ECUDA;
      attr = true;
    }
    int grid = (int)std::min<int64_t>(i1 - i0, (int64_t)num_sms() * 3);
    if (grid < 1) return LEANOT_OK;
    kern<<<grid, RP_THREADS, TAB_BYTES, st>>>(cv, i0, i1, v, sgn, scale, vmin, L);
    return LEANOT_OK;
  }
};

int launch_rowlse(const CostView& cv, int64_t i0, int64_t i1, const double* v, double sgn, double scale, double* L,
                  cudaStream_t st, const double* vmin) {
  RowLseFn f{cv, i0, i1, v, sgn, scale, vmin, L, st};
  return LEANOT_DISPATCH_COST(cv, f);
}

struct RowMinFn {
  const CostView& cv;
  int64_t i0, i1;
  const double* v;
  double* out;
  cudaStream_t st;
  template <class COST>
  int run() {
    int grid = (int)std::min<int64_t>(i1 - i0, (int64_t)num_sms() * 8);
    if (grid < 1) return LEANOT_OK;
    rowmin_kernel<COST><<<grid, RP_THREADS, 0, st>>>(cv, i0, i1, v, out);
    return LEANOT_OK;
  }
};

int launch_rowmin(const CostView& cv, int64_t i0, int64_t i1, const double* v, double* out, cudaStream_t st) {
  RowMinFn f{cv, i0, i1, v, out, st};
  return LEANOT_DISPATCH_COST(cv, f);
}

struct CostBlockFn {
  const CostView& cv;
  int64_t i0, i1;
  double* out;
  int64_t ldo;
  cudaStream_t st;
  template <class COST>
  int run() {
    dim3 grid((unsigned)std::min<int64_t>((cv.n + 255) / 256, 64), (unsigned)std::min<int64_t>(i1 - i0, 4096));
    if (i1 <= i0) return LEANOT_OK;
    cost_block_kernel<COST><<<grid, 256, 0, st>>>(cv, i0, i1, out, ldo);
    return LEANOT_OK;
  }
};

int launch_cost_block(const CostView& cv, int64_t i0, int64_t i1, double* out, int64_t ldo, cudaStream_t st) {
  CostBlockFn f{cv, i0, i1, out, ldo, st};
  return LEANOT_DISPATCH_COST(cv, f);
}

}  // namespace leanot
