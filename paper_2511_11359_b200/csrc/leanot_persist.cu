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
  for (int q = threadIdx.x; q < cnt; q += PS_THREADS) t = fmax(t, p[q]);
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

static bool persist_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LEANOT_PERSIST");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
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
  PersistFn f{A, 2, P.splits, (size_t)(TAB_BYTES + ((n + 1) & ~int64_t(1)) * 8), st};
  return LEANOT_DISPATCH_COST(A.cost, f);
}

}  // namespace leanot
