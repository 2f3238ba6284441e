// Persistent DXG iterations for small single-process plans (n <= 4096; BASELINE config 1).
//
// At n = 1e3 an iteration is ~4e6 exps -- a few microseconds of FP64 work spread over 148 SMs
// -- so the 4-5 launches per iteration of the regular path (pass A, fixup, pass B, slab
// reduce, update) dominate.  Here `iters` whole iterations (dxg_step, dxg.py:261-279) run in
// ONE cooperative kernel, phases separated by grid-wide barriers:
//   pass A   groups of RQ rows per CTA, threads across the columns: S_ki = sum_j
//            exp(x_kij - m_i LSTEP) for both weight sets; out-of-range sums recomputed with an
//            exact row max (same rule as fixup_kernel); finalize as finalize_row (S, shift
//            used, g*EC coefficients, next-iteration shift)
//   pass B   32-column tiles x row splits, lanes over columns, per-row constants staged in
//            shared memory: slab[split][k][j]
//   update 1 fixed-order slab reduce -> col; dual_md_step / balance / b' (dxg.py:223-258)
//   update 2 b = b' - max b', sd, b_bar' (+ a, a_bar, s, t)
//   b_bar    b_bar = b_bar' - max b_bar' (every CTA keeps the full vector in shared memory)
// Same arithmetic per element as the regular kernels; every reduction has a fixed order
// (deterministic).  Evaluation sweeps stay on the regular path.  Included by leanot_lib.cu.
#include <cooperative_groups.h>

namespace leanot {

namespace cg = cooperative_groups;

constexpr int PS_THREADS = 256;
constexpr int PS_WARPS = PS_THREADS / 32;
constexpr int64_t PS_MAX_N = 4096;
constexpr int RQ = 4;   // pass A: rows per CTA group
constexpr int JU = 4;   // pass A: columns per thread in flight (per row of the group)
constexpr int QU = 16;  // pass B: rows per warp in flight

struct PersistArgs {
  CostView cost;
  UpdArgs U;        // O(n) state, scalars and update constants (make_upd)
  const double* r;  // row marginal
  int64_t* shift;   // n: row shift for the next iteration
  int64_t* m;       // 2 x n: shift used per weight set
  double* S;        // 2 x n
  double* coef;     // 2 x n x 4
  double* slab;     // splits x 2 x n
  double* gmax;     // 2 x gridDim.x block maxima
  int splits, ntile, iters;
  int64_t rows_per;  // pass B rows per split
  // row-owner kernel only: start from the marginals in U.col (the last sweep of the state),
  // and/or finish with an evaluation sweep of the final state (evalbuf as leanot_dxg_eval)
  int start_update, eval;
  double eta;
  double* evalbuf;
  double* epart;     // gridDim.x x 5 per-CTA evaluation partials
};

__device__ __forceinline__ double block_max_bcast(double v, double* red) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = red[0];
#pragma unroll
  for (int w = 1; w < PS_WARPS; ++w) t = fmax(t, red[w]);
  __syncthreads();
  return t;
}

__device__ __forceinline__ double block_sum_bcast(double v, double* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = red[0];
#pragma unroll
  for (int w = 1; w < PS_WARPS; ++w) t += red[w];
  __syncthreads();
  return t;
}

// max of cnt block maxima, loaded in parallel by the block (max is order-independent)
__device__ __forceinline__ double max_over(const double* p, int cnt, double* red) {
  double t = -INFINITY;
  for (int q = threadIdx.x; q < cnt; q += PS_THREADS) t = fmax(t, __ldcg(p + q));  // written by other CTAs
  return block_max_bcast(t, red);
}

template <class COST>
__global__ void __launch_bounds__(PS_THREADS) dxg_persist_kernel(const PersistArgs P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) char smem[];
  double* sbb = reinterpret_cast<double*>(smem + TAB_BYTES);  // b_bar, all n
  double* scoef = sbb + ((P.U.n + 1) & ~int64_t(1));          // pass B: rows_per x 8 constants (16 B aligned)
  uint32_t* sm = reinterpret_cast<uint32_t*>(scoef + P.rows_per * 8);  // pass B: rows_per x 2 shifts
  __shared__ double red[PS_WARPS];
  __shared__ double cred[PS_WARPS][2][32];
  __shared__ double pred[PS_WARPS][2 * RQ];
  __shared__ double sS[2 * RQ];
  __shared__ int64_t smk[2 * RQ];
  load_table(reinterpret_cast<double*>(smem));
  const UpdArgs& U = P.U;
  const int64_t n = U.n;
  const int G = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gtid = (int64_t)blockIdx.x * PS_THREADS + threadIdx.x, gthreads = (int64_t)G * PS_THREADS;
  for (int64_t j = threadIdx.x; j < n; j += PS_THREADS) sbb[j] = U.b_bar[j];
  __syncthreads();
  const uint32_t tb = lane_tab_addr(smem);
  const COST cost(P.cost);

  for (int it = 0; it < P.iters; ++it) {
    const double na[2] = {-U.scal[0], -U.scal[1]};
    // ---- pass A: rows blockIdx.x + G q, RQ rows at a time; all threads sweep the columns of
    //      the group with every load of a round in flight, then a fixed-order block reduce
    for (int64_t ib = blockIdx.x; ib < n; ib += (int64_t)G * RQ) {
      typename COST::Row rows[RQ];
      uint32_t mlo[RQ];
#pragma unroll
      for (int q = 0; q < RQ; ++q) {
        const int64_t i = ib + (int64_t)G * q < n ? ib + (int64_t)G * q : ib;
        rows[q] = cost.row(i);
        mlo[q] = (uint32_t)P.shift[i];
      }
      if (threadIdx.x < 2 * RQ) {
        const int64_t i = ib + (int64_t)G * (threadIdx.x >> 1);
        smk[threadIdx.x] = i < n ? P.shift[i] : 0;
      }
      double s[RQ][2];
#pragma unroll
      for (int q = 0; q < RQ; ++q) s[q][0] = s[q][1] = 0.0;
      for (int64_t j0 = threadIdx.x; j0 < n; j0 += (int64_t)PS_THREADS * JU) {
        double c[RQ][JU], nb0[JU], nb1[JU];
#pragma unroll
        for (int u = 0; u < JU; ++u) {
          const int64_t j = j0 + (int64_t)PS_THREADS * u;
          const int64_t jj = j < n ? j : 0;
          nb0[u] = -U.b[jj];
          nb1[u] = -sbb[jj];
#pragma unroll
          for (int q = 0; q < RQ; ++q) c[q][u] = cost.eval1(rows[q], jj);
        }
#pragma unroll
        for (int u = 0; u < JU; ++u) {
          if (j0 + (int64_t)PS_THREADS * u < n) {
#pragma unroll
            for (int q = 0; q < RQ; ++q) {
              texp_acc(tb, fma(na[0], c[q][u], nb0[u]), mlo[q], s[q][0]);
              texp_acc(tb, fma(na[1], c[q][u], nb1[u]), mlo[q], s[q][1]);
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < RQ; ++q)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const double v = warp_sum(s[q][k]);
          if (lane == 0) pred[warp][q * 2 + k] = v;
        }
      __syncthreads();
      if (threadIdx.x < 2 * RQ) {
        double t = pred[0][threadIdx.x];
#pragma unroll
        for (int w = 1; w < PS_WARPS; ++w) t += pred[w][threadIdx.x];
        sS[threadIdx.x] = t;
      }
      __syncthreads();
      // sums outside [2^-900, 2^900]: recompute that row with an exact max shift (fixup_kernel)
      for (int v = 0; v < 2 * RQ; ++v) {
        const int q = v >> 1, k = v & 1;
        if (ib + (int64_t)G * q >= n || sum_ok(sS[v])) continue;  // block-uniform
        double mx = -INFINITY;
        for (int64_t j = threadIdx.x; j < n; j += PS_THREADS)
          mx = fmax(mx, fma(na[k], cost.eval1(rows[q], j), -(k == 0 ? U.b[j] : sbb[j])));
        mx = block_max_bcast(mx, red);
        const int64_t m = llrint(mx * (1.0 / LSTEP));
        double t = 0.0;
        for (int64_t j = threadIdx.x; j < n; j += PS_THREADS)
          texp_acc(tb, fma(na[k], cost.eval1(rows[q], j), -(k == 0 ? U.b[j] : sbb[j])), (uint32_t)m, t);
        t = block_sum_bcast(t, red);
        if (threadIdx.x == 0) {
          sS[v] = t;
          smk[v] = m;
        }
        __syncthreads();
      }
      // finalize_row for both weight sets of each row of the group
      if (threadIdx.x < RQ) {
        const int q = threadIdx.x;
        const int64_t i = ib + (int64_t)G * q;
        if (i < n) {
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const double Sk = sS[2 * q + k];
            P.S[k * n + i] = Sk;
            P.m[k * n + i] = smk[2 * q + k];
            const double g = P.r[i] / Sk;
            double* cf = P.coef + (k * n + i) * 4;
            cf[0] = g * EC0; cf[1] = g * EC1; cf[2] = g * EC2; cf[3] = g * EC3;
          }
          // next-iteration shift from the midpoint weight set (make_rowpass: next_from_k = 1)
          P.shift[i] = smk[2 * q + 1] + llrint(log(sS[2 * q + 1]) * (1.0 / LSTEP));
        }
      }
      __syncthreads();
    }
    grid.sync();
    // ---- pass B: (32-column tile, row split) per CTA, lanes over columns, warps over rows
    const int64_t rows_per = P.rows_per;
    for (int item = blockIdx.x; item < P.ntile * P.splits; item += G) {
      const int tile = item % P.ntile, split = item / P.ntile;
      const int64_t j = (int64_t)tile * 32 + lane;
      const bool valid = j < n;
      const int64_t jj = valid ? j : 0;
      const double nb0 = valid ? -U.b[j] : 0.0, nb1 = valid ? -sbb[j] : 0.0;
      const int64_t r0 = split * rows_per, r1 = r0 + rows_per < n ? r0 + rows_per : n;
      // the item's per-row constants (g*EC for both sets, shifts) staged in one coalesced round
      const int nrow = (int)(r1 - r0);
      for (int e = threadIdx.x; e < nrow * 8; e += PS_THREADS) {
        const int q = e >> 3, c = e & 7;
        scoef[e] = P.coef[((c >> 2) * n + r0 + q) * 4 + (c & 3)];
      }
      for (int e = threadIdx.x; e < nrow * 2; e += PS_THREADS)
        sm[e] = (uint32_t)P.m[(e & 1) * n + r0 + (e >> 1)];
      __syncthreads();
      double acc0 = 0.0, acc1 = 0.0;
      // QU rows per warp per step: the C loads of the step first, constants from shared memory
      for (int64_t i0 = r0 + warp; i0 < r1; i0 += PS_WARPS * QU) {
        double c[QU];
#pragma unroll
        for (int u = 0; u < QU; ++u) {
          const int64_t i = i0 + (int64_t)PS_WARPS * u < r1 ? i0 + (int64_t)PS_WARPS * u : r1 - 1;
          c[u] = cost.eval1(cost.row(i), jj);
        }
#pragma unroll
        for (int u = 0; u < QU; ++u) {
          const int64_t i = i0 + (int64_t)PS_WARPS * u;
          if (i < r1) {
            const double2* cq = reinterpret_cast<const double2*>(scoef + (i - r0) * 8);
            const double2 a01 = cq[0], a23 = cq[1], b01 = cq[2], b23 = cq[3];
            texp_gacc(tb, fma(na[0], c[u], nb0), sm[(i - r0) * 2], a01.x, a01.y, a23.x, a23.y, acc0);
            texp_gacc(tb, fma(na[1], c[u], nb1), sm[(i - r0) * 2 + 1], b01.x, b01.y, b23.x, b23.y, acc1);
          }
        }
      }
      cred[warp][0][lane] = acc0;
      cred[warp][1][lane] = acc1;
      __syncthreads();
      if (warp < 2 && valid) {
        double v = cred[0][warp][lane];
#pragma unroll
        for (int w = 1; w < PS_WARPS; ++w) v += cred[w][warp][lane];
        P.slab[((int64_t)split * 2 + warp) * n + j] = v;
      }
      __syncthreads();
    }
    grid.sync();
    // ---- update 1: columns, mirror steps, b' (dxg_update_small, first loop)
    double mx = -INFINITY;
    for (int64_t j = gtid; j < n; j += gthreads) {
      // fixed-order sum over the splits, loads of 8 splits in flight at a time
      double cn = 0.0, cb = 0.0;
      for (int q0 = 0; q0 < P.splits; q0 += 8) {
        double vn[8], vb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int q = q0 + u < P.splits ? q0 + u : q0;
          vn[u] = P.slab[(int64_t)(2 * q) * n + j];
          vb[u] = P.slab[(int64_t)(2 * q + 1) * n + j];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (q0 + u < P.splits) { cn += vn[u]; cb += vb[u]; }
      }
      const_cast<double*>(U.col)[j] = cn;
      const_cast<double*>(U.col)[n + j] = cb;
      const double cj = U.c[j], ctj = U.ct[j], dj = U.delta[j];
      const double dbar = md_step(U.A, U.B, dj, cn, cj, ctj);
      double dn = md_step(U.A, U.B, dj, cb, cj, ctj);
      dn = fmin(fmax(dn, -U.beta), U.beta);
      const double bp = __dadd_rn(__dmul_rn(U.decay, U.b[j]), __dmul_rn(U.G, tanh(__dmul_rn(0.5, dbar))));
      U.delta[j] = dn;
      U.bprime[j] = bp;
      mx = fmax(mx, bp);
    }
    mx = block_max_bcast(mx, red);
    if (threadIdx.x == 0) P.gmax[blockIdx.x] = mx;
    grid.sync();
    // ---- update 2: b = b' - max b', sd, b_bar'
    {
      const double M = max_over(P.gmax, G, red);
      double mb = -INFINITY;
      for (int64_t j = gtid; j < n; j += gthreads) {
        const double bn = __dsub_rn(U.bprime[j], M);
        const double d = tanh(__dmul_rn(0.5, U.delta[j]));
        const double bb = __dadd_rn(__dmul_rn(U.decay, bn), __dmul_rn(U.G, d));
        U.b[j] = bn;
        U.sd[j] = __dmul_rn(U.twosup, d);
        U.bprime[j] = bb;
        mb = fmax(mb, bb);
      }
      mb = block_max_bcast(mb, red);
      if (threadIdx.x == 0) P.gmax[G + blockIdx.x] = mb;
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        const double a = __dadd_rn(__dmul_rn(U.decay, U.scal[0]), U.tau_p);
        U.scal[0] = a;
        U.scal[1] = __dadd_rn(__dmul_rn(U.decay, a), U.tau_p);
        U.scal[2] = __dadd_rn(__dmul_rn(U.decay, U.scal[2]), U.tau_p_eta);
        U.scal[3] = U.scal[3] + 1.0;
      }
    }
    grid.sync();
    // ---- b_bar = b_bar' - max b_bar': shared copy in every CTA, global copy for the host
    {
      const double Mb = max_over(P.gmax + G, G, red);
      for (int64_t j = threadIdx.x; j < n; j += PS_THREADS) sbb[j] = __dsub_rn(U.bprime[j], Mb);
      for (int64_t j = gtid; j < n; j += gthreads) U.b_bar[j] = __dsub_rn(U.bprime[j], Mb);
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------------------
// Row-owner persistent iterations for n <= 1024 (BASELINE config 1): the single-read form.
// CTA c owns rows [c R, c R + R) (R = ceil(n / G) <= 8) and keeps their exps in registers
// (256 threads x 4 columns x R rows x 2 weight sets), so pass B is an FMA over the stored
// exps instead of a second exp and needs no grid barrier after pass A (the row sums are
// CTA-local).  Per iteration two grid barriers instead of four:
//   A+B (own rows) -> slab[c][k][j] | sync | column owners: fixed-order sum of the G partials,
//   dual_md_step / balance / b' (dxg.py:223-258), block max | sync | every CTA: b, sd, b_bar'
//   for all n columns (redundant, bitwise identical), max b_bar' locally, b_bar in shared
//   memory; owners write the state back.  Same per-element arithmetic (table exp, shifts from
//   the previous iteration, exact-max recompute of out-of-range rows) and fixed reduction
//   orders; the column sums are sum_i g_i e_ij with the product formed after the exp
//   (the regular pass B folds g into the polynomial: same value to a few ulps).
constexpr int PO_THREADS = 256;            // 8 warps, 255-register budget for the exps held in registers
constexpr int PO_WARPS = PO_THREADS / 32;
constexpr int PO_J = 4;                    // columns per thread (n <= 1024)
constexpr int PO_R = 8;                    // max rows per CTA
constexpr int64_t PO_MAX_N = PO_THREADS * PO_J;
constexpr int PO_LPV = PO_THREADS / 16;    // lanes per value in the column sums (16 values)
constexpr int PO_PARTS = 12;               // partials per lane in the column sums (G <= 192)

__device__ __forceinline__ double po_block_max(double v, double* red) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = red[0];
#pragma unroll
  for (int w = 1; w < PO_WARPS; ++w) t = fmax(t, red[w]);
  __syncthreads();
  return t;
}
__device__ __forceinline__ double po_block_sum(double v, double* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = red[0];
#pragma unroll
  for (int w = 1; w < PO_WARPS; ++w) t += red[w];
  __syncthreads();
  return t;
}
__device__ __forceinline__ double po_max_over(const double* p, int cnt, double* red) {
  double t = -INFINITY;
  for (int q = threadIdx.x; q < cnt; q += PO_THREADS) t = fmax(t, __ldcg(p + q));  // written by other CTAs
  return po_block_max(t, red);
}

#ifdef LEANOT_DBG_TIMING
#define PO_TS(slot)                                                                     \
  do {                                                                                  \
    if (blockIdx.x == 0 && threadIdx.x == 0 && it == 5) {                               \
      uint64_t t_;                                                                      \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
      reinterpret_cast<uint64_t*>(const_cast<double*>(P.U.partial))[slot] = t_;         \
    }                                                                                   \
  } while (0)
#else
#define PO_TS(slot) do {} while (0)
#endif

template <class COST>
__global__ void __launch_bounds__(PO_THREADS, 1) dxg_rowowner_kernel(const PersistArgs P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) char smem[];
  const UpdArgs& U = P.U;
  const int64_t n = U.n;
  double* sb = reinterpret_cast<double*>(smem + TAB_BYTES);  // b, all n
  double* sbb = sb + PO_MAX_N;                                // b_bar, all n
  double* sC = sbb + PO_MAX_N;                                // own rows of C [PO_R][n] (constant)
  __shared__ double red[PO_WARPS];
  __shared__ double pred[PO_WARPS][2 * PO_R];
  __shared__ double sS[2 * PO_R], sg[2 * PO_R];
  __shared__ int64_t smk[2 * PO_R];
  __shared__ double scol[32];
  load_table(reinterpret_cast<double*>(smem));
  const int G = gridDim.x, c = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t j = threadIdx.x; j < n; j += PO_THREADS) { sb[j] = U.b[j]; sbb[j] = U.b_bar[j]; }
  double sc[4];  // a, a_bar, s, t (every CTA advances its own copy; CTA 0 publishes)
#pragma unroll
  for (int q = 0; q < 4; ++q) sc[q] = U.scal[q];
  __syncthreads();
  const uint32_t tb = lane_tab_addr(smem);
  const COST cost(P.cost);
  const int rpc = (int)((n + G - 1) / G);
  const int64_t i0 = (int64_t)c * rpc;
  const int nrow = (int)(i0 >= n ? 0 : (n - i0 < rpc ? n - i0 : rpc));
  const int grows = (int)((n + rpc - 1) / rpc);  // CTAs that own rows
  const int cpc = rpc;                           // columns owned per CTA (same split)
  const int64_t j0c = (int64_t)c * cpc;
  const int ncol = (int)(j0c >= n ? 0 : (n - j0c < cpc ? n - j0c : cpc));
  // the own rows' costs stay in shared memory for the whole launch (pass A reads them with
  // LDS latency instead of one dependent global load per element)
  for (int q = 0; q < nrow; ++q) {
    const typename COST::Row rq = cost.row(i0 + q);
    for (int64_t j = threadIdx.x; j < n; j += PO_THREADS) sC[q * n + j] = cost.eval1(rq, j);
  }
  double rw[PO_R];
#pragma unroll
  for (int q = 0; q < PO_R; ++q) rw[q] = q < nrow ? P.r[i0 + q] : 0.0;
  // owner threads keep their column's marginal constants and dual in registers (only the
  // owner writes delta_j; everybody else reads it after the second barrier)
  const bool owner = threadIdx.x < ncol;
  const int64_t jo = owner ? j0c + threadIdx.x : 0;
  const double c_o = owner ? U.c[jo] : 0.0, ct_o = owner ? U.ct[jo] : 1.0;
  double d_o = owner ? U.delta[jo] : 0.0;
  __syncthreads();

  for (int it = 0; it <= P.iters; ++it) {
    const bool last = it == P.iters;  // the evaluation sweep of the final state (if requested)
    if (last && !P.eval) break;
    const double na[2] = {-sc[0], -sc[1]};
    double cn_o = 0.0, cb_o = 0.0;    // owner: the column's two marginals
    if (it == 0 && P.start_update) {
      if (owner) { cn_o = U.col[jo]; cb_o = U.col[n + jo]; }
    } else {
    PO_TS(0);
    // ---- pass A on the own rows; exps kept in registers ----
    double e[PO_R][PO_J][2], s[PO_R][2];
    uint32_t mlo[PO_R];
    int64_t msh[PO_R];
#pragma unroll
    for (int q = 0; q < PO_R; ++q) {
      msh[q] = q < nrow ? P.shift[i0 + q] : 0;
      mlo[q] = (uint32_t)msh[q];
      s[q][0] = s[q][1] = 0.0;
    }
#pragma unroll
    for (int u = 0; u < PO_J; ++u) {
      const int64_t j = threadIdx.x + (int64_t)PO_THREADS * u;
      const bool valid = j < n;
      const int64_t jj = valid ? j : 0;
      const double nb0 = -sb[jj], nb1 = -sbb[jj];
#pragma unroll
      for (int q = 0; q < PO_R; ++q) {
        // rows q >= nrow / columns j >= n compute on a valid (unused) operand and are masked
        const double cq = sC[(q < nrow ? q : 0) * n + jj];
        const bool on = q < nrow && valid;
        const double e0 = texp(tb, fma(na[0], cq, nb0), mlo[q]);
        const double e1 = texp(tb, fma(na[1], cq, nb1), mlo[q]);
        e[q][u][0] = on ? e0 : 0.0;
        e[q][u][1] = on ? e1 : 0.0;
        s[q][0] += e[q][u][0];
        s[q][1] += e[q][u][1];
      }
    }
    // block sums of the 2 R row sums: per-warp transpose-reduce (value (lane >> 1) & 15 on
    // even lanes), then the warps in order
    {
      double v8[8], v4[4], v2[2];
      const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double lo = s[i >> 1][i & 1], hi = s[(i + 8) >> 1][(i + 8) & 1];
        v8[i] = (b4 ? hi : lo) + __shfl_xor_sync(0xffffffffu, b4 ? lo : hi, 16);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        v4[i] = (b3 ? v8[i + 4] : v8[i]) + __shfl_xor_sync(0xffffffffu, b3 ? v8[i] : v8[i + 4], 8);
#pragma unroll
      for (int i = 0; i < 2; ++i)
        v2[i] = (b2 ? v4[i + 2] : v4[i]) + __shfl_xor_sync(0xffffffffu, b2 ? v4[i] : v4[i + 2], 4);
      double x = (b1 ? v2[1] : v2[0]) + __shfl_xor_sync(0xffffffffu, b1 ? v2[0] : v2[1], 2);
      x += __shfl_xor_sync(0xffffffffu, x, 1);
      if ((lane & 1) == 0) pred[warp][(lane >> 1) & 15] = x;
    }
    PO_TS(1);
    __syncthreads();
    if (threadIdx.x < 2 * PO_R) {
      double t = pred[0][threadIdx.x];
#pragma unroll
      for (int w = 1; w < PO_WARPS; ++w) t += pred[w][threadIdx.x];
      sS[threadIdx.x] = t;
    }
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 0; q < PO_R; ++q) smk[2 * q] = smk[2 * q + 1] = msh[q];
    }
    __syncthreads();
    // out-of-range sums: exact max shift for that row and weight set, exps recomputed
#pragma unroll
    for (int q = 0; q < PO_R; ++q)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (q >= nrow || sum_ok(sS[2 * q + k])) continue;  // block-uniform
        const double* bk = k == 0 ? sb : sbb;
        const double* cr = sC + q * n;
        double mx = -INFINITY;
        for (int64_t j = threadIdx.x; j < n; j += PO_THREADS) mx = fmax(mx, fma(na[k], cr[j], -bk[j]));
        mx = po_block_max(mx, red);
        const int64_t m = llrint(mx * (1.0 / LSTEP));
        double t = 0.0;
#pragma unroll
        for (int u = 0; u < PO_J; ++u) {
          const int64_t j = threadIdx.x + (int64_t)PO_THREADS * u;
          e[q][u][k] = j < n ? texp(tb, fma(na[k], cr[j], -bk[j]), (uint32_t)m) : 0.0;
          t += e[q][u][k];
        }
        t = po_block_sum(t, red);
        if (threadIdx.x == 0) {
          sS[2 * q + k] = t;
          smk[2 * q + k] = m;
        }
        __syncthreads();
      }
    // finalize the own rows (dxg outputs, next-iteration shift from the midpoint set)
    if (threadIdx.x < 2 * PO_R) {
      const int q = threadIdx.x >> 1, k = threadIdx.x & 1;
      if (q < nrow) {
        const int64_t i = i0 + q;
        const double Sk = sS[threadIdx.x];
        P.S[k * n + i] = Sk;
        P.m[k * n + i] = smk[threadIdx.x];
        double rq = rw[0];
#pragma unroll
        for (int qq = 1; qq < PO_R; ++qq) rq = q == qq ? rw[qq] : rq;
        sg[threadIdx.x] = rq / Sk;
        if (k == 1) P.shift[i] = smk[threadIdx.x] + llrint(log(Sk) * (1.0 / LSTEP));
      } else {
        sg[threadIdx.x] = 0.0;
      }
    }
    __syncthreads();
    PO_TS(2);
    // ---- pass B on the own rows: column partials from the stored exps ----
#pragma unroll
    for (int u = 0; u < PO_J; ++u) {
      const int64_t j = threadIdx.x + (int64_t)PO_THREADS * u;
      if (j < n && c < grows) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int q = 0; q < PO_R; ++q) {
          a0 = fma(sg[2 * q], e[q][u][0], a0);
          a1 = fma(sg[2 * q + 1], e[q][u][1], a1);
        }
        P.slab[((int64_t)c * 2) * n + j] = a0;
        P.slab[((int64_t)c * 2 + 1) * n + j] = a1;
      }
    }
    if (last) {  // after pass B: the register-resident exps are dead here
      // evaluation statistics of weight set 0 over the own rows (rowpass EVAL + eval kernels):
      // <C, D_r p>, sum_i r_i H(p_i) and sum_i r_i v_i with v_i = min_j (C_ij + sd_j) (eta = 0,
      // dxg.py:344-348) or LSE_j(-(C_ij + sd_j) / eta) (dxg.py:337); fixed orders
      double rs0 = 0.0, rs1 = 0.0, rs2 = 0.0;
#pragma unroll 1
      for (int q = 0; q < nrow; ++q) {  // block-uniform
        // the exps of weight set 0 recomputed with the shift pass A used (bitwise the same
        // values; keeps the register-resident e[][][] statically indexed)
        const uint32_t m0 = (uint32_t)smk[2 * q];
        double uu = 0.0, vv = 0.0, mn = INFINITY;
        for (int64_t j = threadIdx.x; j < n; j += PO_THREADS) {
          const double cq = sC[q * n + j];
          const double x0 = fma(na[0], cq, -sb[j]);
          const double e0 = texp(tb, x0, m0);
          uu = fma(e0, cq, uu);
          vv = fma(e0, x0, vv);
          mn = fmin(mn, cq + __ldcg(U.sd + j));
        }
        uu = po_block_sum(uu, red);
        vv = po_block_sum(vv, red);
        double v;
        if (P.eta > 0) {
          const double ie = -1.0 / P.eta;
          double mx = -INFINITY;
          for (int64_t j = threadIdx.x; j < n; j += PO_THREADS) mx = fmax(mx, (sC[q * n + j] + __ldcg(U.sd + j)) * ie);
          mx = po_block_max(mx, red);
          double t = 0.0;
          for (int64_t j = threadIdx.x; j < n; j += PO_THREADS) t += exp((sC[q * n + j] + __ldcg(U.sd + j)) * ie - mx);
          t = po_block_sum(t, red);
          v = mx + log(t);
        } else {
          v = po_block_max(-mn, red);
          v = -v;
        }
        double rq = rw[0];
#pragma unroll
        for (int qq = 1; qq < PO_R; ++qq) rq = q == qq ? rw[qq] : rq;
        const double S0 = sS[2 * q];
        rs0 += (rq / S0) * uu;
        if (rq > 0.0) rs1 += rq * (((double)smk[2 * q] * LSTEP + log(S0)) - vv / S0);
        rs2 += rq * v;
      }
      if (threadIdx.x == 0) {
        P.epart[c * 5 + 0] = rs0;
        P.epart[c * 5 + 1] = rs1;
        P.epart[c * 5 + 2] = rs2;
      }
    }
    PO_TS(3);
    grid.sync();
    PO_TS(4);
    // ---- owned columns: fixed-order sum of the partials (16 lanes per value), updates ----
    {
      const int v = threadIdx.x / PO_LPV, part = threadIdx.x % PO_LPV;  // value v = 2 * column + set
      double t = 0.0;
      if (v < 2 * ncol) {
        // all of this lane's partials in flight at once, then added in order
        const int64_t j = j0c + (v >> 1);
        double pv[PO_PARTS];
#pragma unroll
        for (int u = 0; u < PO_PARTS; ++u) {
          const int p = part + PO_LPV * u;
          pv[u] = p < grows ? __ldcg(P.slab + ((int64_t)p * 2 + (v & 1)) * n + j) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PO_PARTS; ++u) t += pv[u];
      }
#pragma unroll
      for (int o = PO_LPV / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (part == 0 && v < 16) scol[v] = t;
    }
    __syncthreads();
    if (owner) {
      cn_o = scol[2 * threadIdx.x];
      cb_o = scol[2 * threadIdx.x + 1];
      const_cast<double*>(U.col)[jo] = cn_o;
      const_cast<double*>(U.col)[n + jo] = cb_o;
    }
    }  // sweep of this step
    if (last) {
      // column statistics of the swept state (colstats_reduce_kernel), then the fixed-order
      // combination of the per-CTA partials by CTA 0
      double s3 = owner ? fabs(cn_o - c_o) : 0.0;
      double s4 = owner ? c_o * tanh(0.5 * d_o) : 0.0;
      s3 = po_block_sum(s3, red);
      s4 = po_block_sum(s4, red);
      if (threadIdx.x == 0) {
        P.epart[c * 5 + 3] = s3;
        P.epart[c * 5 + 4] = s4;
      }
      grid.sync();
      if (c == 0 && threadIdx.x < 5) {
        double t = 0.0;
        for (int q = 0; q < G; ++q) t += __ldcg(P.epart + q * 5 + threadIdx.x);
        P.evalbuf[threadIdx.x] = t;
      }
      if (c == 0 && threadIdx.x < 4) P.evalbuf[8 + threadIdx.x] = sc[threadIdx.x];
      break;
    }
    double mx = -INFINITY;
    if (owner) {
      const int64_t j = jo;
      const double cn = cn_o, cb = cb_o;
      const double dbar = md_step(U.A, U.B, d_o, cn, c_o, ct_o);
      double dn = md_step(U.A, U.B, d_o, cb, c_o, ct_o);
      dn = fmin(fmax(dn, -U.beta), U.beta);
      const double bp = __dadd_rn(__dmul_rn(U.decay, sb[j]), __dmul_rn(U.G, tanh(__dmul_rn(0.5, dbar))));
      d_o = dn;
      U.delta[j] = dn;
      U.bprime[j] = bp;
      mx = bp;
    }
    mx = po_block_max(mx, red);
    if (threadIdx.x == 0) P.gmax[c] = mx;
    PO_TS(5);
    grid.sync();
    PO_TS(6);
    // ---- every CTA: b = b' - max b', sd, b_bar' for all columns; b_bar = b_bar' - max ----
    {
      // loads of b' and delta first (independent of the max), so both latencies overlap
      double bpv[PO_J], dv[PO_J];
#pragma unroll
      for (int u = 0; u < PO_J; ++u) {
        const int64_t j = threadIdx.x + (int64_t)PO_THREADS * u;
        bpv[u] = j < n ? __ldcg(U.bprime + j) : 0.0;
        dv[u] = j < n ? tanh(__dmul_rn(0.5, __ldcg(U.delta + j))) : 0.0;
      }
      const double M = po_max_over(P.gmax, G, red);
      double mb = -INFINITY;
#pragma unroll
      for (int u = 0; u < PO_J; ++u) {
        const int64_t j = threadIdx.x + (int64_t)PO_THREADS * u;
        if (j < n) {
          const double bn = __dsub_rn(bpv[u], M);
          const double d = dv[u];
          const double bb = __dadd_rn(__dmul_rn(U.decay, bn), __dmul_rn(U.G, d));
          sb[j] = bn;
          sbb[j] = bb;
          mb = fmax(mb, bb);
          if (j >= j0c && j < j0c + ncol) {
            U.b[j] = bn;
            U.sd[j] = __dmul_rn(U.twosup, d);
          }
        }
      }
      mb = po_block_max(mb, red);
#pragma unroll
      for (int u = 0; u < PO_J; ++u) {
        const int64_t j = threadIdx.x + (int64_t)PO_THREADS * u;
        if (j < n) {
          const double bb = __dsub_rn(sbb[j], mb);
          sbb[j] = bb;
          if (j >= j0c && j < j0c + ncol) U.b_bar[j] = bb;
        }
      }
      const double a = __dadd_rn(__dmul_rn(U.decay, sc[0]), U.tau_p);
      sc[0] = a;
      sc[1] = __dadd_rn(__dmul_rn(U.decay, a), U.tau_p);
      sc[2] = __dadd_rn(__dmul_rn(U.decay, sc[2]), U.tau_p_eta);
      sc[3] = sc[3] + 1.0;
      __syncthreads();
    }
    PO_TS(7);
  }
  if (c == 0 && threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) U.scal[q] = sc[q];
  }
}

static inline int64_t a_n(const PersistArgs& P) { return P.U.n; }

struct RowOwnerFn {
  const PersistArgs& P;
  int64_t slab_doubles;
  cudaStream_t st;
  template <class COST>
  int run() {
    auto kern = dxg_rowowner_kernel<COST>;
    const size_t smem = TAB_BYTES + 2 * PO_MAX_N * 8 + (size_t)PO_R * a_n(P) * 8;
    // the shared-memory size depends on the plan (cached cost rows): raise the kernel's limit
    // whenever a plan needs more than the largest one so far (a first, smaller plan must not
    // cap later ones -- that made the occupancy query return 0 for a larger n)
    static size_t attr_smem = 0;  // per instantiation
    if (smem > attr_smem) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        set_error("row-owner: shared memory attribute");
        return LEANOT_EINVAL;
      }
      attr_smem = smem;
    }
    PersistArgs a = P;
    const int64_t n = a.U.n;
    const int G = num_sms();
    if ((n + G - 1) / G > PO_R || n > PO_MAX_N || G > PO_LPV * PO_PARTS) {
      set_error("row-owner: n = %lld does not fit %d CTAs", (long long)n, G);
      return LEANOT_EINVAL;
    }
    if ((int64_t)G * 2 * n + 6 * G > slab_doubles) {
      set_error("row-owner: slab of %lld doubles < %lld", (long long)slab_doubles, (long long)(G * 2 * n + 6 * G));
      return LEANOT_EINVAL;
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, PO_THREADS, smem) != cudaSuccess || occ < 1) {
      set_error("row-owner: occupancy query failed (occ %d)", occ);
      return LEANOT_EINVAL;
    }
    a.gmax = a.slab + (int64_t)G * 2 * n;
    a.epart = a.gmax + G;
    void* args[] = {&a};
    const cudaError_t e = cudaLaunchCooperativeKernel((const void*)kern, G, PO_THREADS, args, smem, st);
    if (e != cudaSuccess) {
      cudaGetLastError();
      set_error("row-owner: cooperative launch: %s", cudaGetErrorString(e));
      return LEANOT_EINVAL;
    }
    return LEANOT_OK;
  }
};

struct PersistFn {
  const PersistArgs& P;
  int blocks_per_sm, max_splits;
  size_t smem;
  cudaStream_t st;
  template <class COST>
  int run() {
    auto kern = dxg_persist_kernel<COST>;
    static bool attr = false;  // per instantiation
    if (!attr) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    PersistArgs a = P;
    const int64_t n = a.U.n;
    // grid: 2 CTAs per SM if the shared-memory footprint allows it, else 1
    for (int bps = blocks_per_sm; bps >= 1; --bps) {
      const int G = num_sms() * bps;
      int splits = std::max(1, G / a.ntile);
      splits = (int)std::min<int64_t>({(int64_t)splits, (int64_t)max_splits, n});
      // block maxima live in the slab tail: needs 2G doubles beyond the used splits
      if ((int64_t)(max_splits - splits) * 2 * n < 2 * G) continue;
      const int64_t rows_per = (n + splits - 1) / splits;
      const size_t smem_all = smem + (size_t)rows_per * (8 * 8 + 2 * 4);
      int occ = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, PS_THREADS, smem_all) != cudaSuccess || occ < bps)
        continue;
      a.splits = splits;
      a.rows_per = rows_per;
      a.gmax = a.slab + (int64_t)splits * 2 * n;
      void* args[] = {&a};
      const cudaError_t e = cudaLaunchCooperativeKernel((const void*)kern, G, PS_THREADS, args, smem_all, st);
      if (e != cudaSuccess) {
        cudaGetLastError();
        return LEANOT_EINVAL;  // caller falls back to the regular path
      }
      return LEANOT_OK;
    }
    return LEANOT_EINVAL;
  }
};

// LEANOT_ROWOWNER=0 keeps the four-barrier persistent kernel for n <= 1024 (A/B comparisons)
// read on every call (not cached): tests switch these paths per test with the environment
static bool rowowner_env() {
  const char* e = getenv("LEANOT_ROWOWNER");
  return !(e && e[0] == '0');
}

static bool persist_env() {
  const char* e = getenv("LEANOT_PERSIST");
  return !(e && e[0] == '0');
}

// Runs `iters` iterations persistently when the plan qualifies; returns LEANOT_OK if it did,
// LEANOT_EINVAL if the caller should use the regular path.
static int try_persist_iterate(const leanot_dxg_plan_t& P, int iters, cudaStream_t st) {
  if (!persist_env() || iters < 1 || P.n > PS_MAX_N || P.row0 != 0 || P.row1 != P.n || use_sep(P)) return LEANOT_EINVAL;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return LEANOT_EINVAL;
  const int64_t n = P.n;
  PersistArgs A;
  A.cost = make_view(P.cost);
  A.U = make_upd(P);
  A.r = P.r;
  A.shift = P.shift;
  A.m = P.m;
  A.S = P.S;
  A.coef = P.coef;
  A.slab = P.slab;
  A.gmax = nullptr;  // set at launch (depends on the grid size)
  A.splits = 0;
  A.ntile = (int)((n + 31) / 32);
  A.iters = iters;
  A.start_update = 0; A.eval = 0; A.eta = P.prm.eta; A.evalbuf = P.evalbuf; A.epart = nullptr;
  if (n <= PO_MAX_N && rowowner_env()) {
    RowOwnerFn g{A, (int64_t)P.splits * 2 * n, st};
    if (LEANOT_DISPATCH_COST(A.cost, g) == LEANOT_OK) return LEANOT_OK;
  }
  PersistFn f{A, 2, P.splits, (size_t)(TAB_BYTES + ((n + 1) & ~int64_t(1)) * 8), st};
  return LEANOT_DISPATCH_COST(A.cost, f);
}

// Interval of solve() (dxg.py:420-472) between two logging points in ONE launch:
// [update from the marginals in U.col when start_update] + the remaining of `iters` updates
// as full iterations + the evaluation sweep of the final state (evalbuf[0..4] as
// leanot_dxg_eval, evalbuf[8..11] = a, a_bar, s, t; U.col = its marginals).  Row-owner
// plans only (single process, n <= 1024, not the separable path); LEANOT_EINVAL otherwise.
static int try_rowowner_iterate_eval(const leanot_dxg_plan_t& P, int iters, int start_update, cudaStream_t st) {
  if (!persist_env() || !rowowner_env() || iters < 0 || P.n > PO_MAX_N || P.row0 != 0 || P.row1 != P.n ||
      use_sep(P))
    return LEANOT_EINVAL;
  if (iters == 0 && start_update) return LEANOT_EINVAL;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return LEANOT_EINVAL;
  const int64_t n = P.n;
  PersistArgs A;
  memset(&A, 0, sizeof(A));
  A.cost = make_view(P.cost);
  A.U = make_upd(P);
  A.r = P.r; A.shift = P.shift; A.m = P.m; A.S = P.S; A.coef = P.coef; A.slab = P.slab;
  A.ntile = (int)((n + 31) / 32);
  A.iters = iters;
  A.start_update = start_update; A.eval = 1; A.eta = P.prm.eta; A.evalbuf = P.evalbuf;
  RowOwnerFn g{A, (int64_t)P.splits * 2 * n, st};
  return LEANOT_DISPATCH_COST(A.cost, g);
}

}  // namespace leanot
