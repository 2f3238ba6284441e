// Dense post-processing for n <= dense cap:
//   - implicit plan materialization D_r p          (materialize_plan, dxg.py:211-220)
//   - Alg. 1 Round onto Pi(r, c)                    (round_to_polytope, rounding.py:63-87)
//   - <C, pi> reductions                           (rounded_cost, dxg.py:471)
// All on a row-major n x n device matrix (leading dimension ld).
// Included by leanot_lib.cu (single translation unit).

namespace leanot {

// P_ij = r_i exp(-(a C_ij + b_j) - L_i)
template <class COST>
__global__ void plan_kernel(const CostView cv, double a, const double* b, const double* r, const double* L, double* P,
                            int64_t ld) {
  const COST cost(cv);
  const int64_t n = cv.n;
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y) {
    const typename COST::Row row = cost.row(i);
    const double ri = r[i], Li = L[i];
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
      P[i * ld + j] = ri * exp(-(a * cost.eval1(row, j) + b[j]) - Li);
  }
}

// row scaling: x_i = min(r_i / row_i, 1) (1 if row_i == 0); m_i* *= x_i  (rounding.py:73-76)
__global__ void round_rows_kernel(double* m, int64_t n, int64_t ld, const double* r) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    double s = 0.0;
    for (int64_t j = lane; j < n; j += 32) s += m[i * ld + j];
    s = warp_sum(s);
    const double x = s > 0 ? fmin(r[i] / s, 1.0) : 1.0;
    for (int64_t j = lane; j < n; j += 32) m[i * ld + j] *= x;
  }
}

// column scaling: y_j = min(c_j / col_j, 1) (1 if col_j == 0); m_*j *= y_j  (rounding.py:77-80)
__global__ void round_cols_kernel(double* m, int64_t n, int64_t ld, const double* c) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += m[i * ld + j];
    const double y = s > 0 ? fmin(c[j] / s, 1.0) : 1.0;
    for (int64_t i = 0; i < n; ++i) m[i * ld + j] *= y;
  }
}

// missing mass: dr_i = max(r_i - rowsum_i, 0), dc_j = max(c_j - colsum_j, 0) (rounding.py:82-83; clamp: see
// rounding.py docstring in the Python layer)
__global__ void round_deficit_rows_kernel(const double* m, int64_t n, int64_t ld, const double* r, double* dr) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    double s = 0.0;
    for (int64_t j = lane; j < n; j += 32) s += m[i * ld + j];
    s = warp_sum(s);
    if (lane == 0) dr[i] = fmax(r[i] - s, 0.0);
  }
}

__global__ void round_deficit_cols_kernel(const double* m, int64_t n, int64_t ld, const double* c, double* dc) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += m[i * ld + j];
    dc[j] = fmax(c[j] - s, 0.0);
  }
}

__global__ void sum_kernel(const double* v, int64_t n, double* out) {
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
  s = block_sum(s);
  if (threadIdx.x == 0) out[0] = s;
}

// m += dr dc^T / mass when mass > 1e-15 (rounding.py:84-86); mass read on device
__global__ void round_outer_kernel(double* m, int64_t n, int64_t ld, const double* dr, const double* dc,
                                   const double* mass) {
  const double ms = *mass;
  if (!(ms > 1e-15)) return;
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y) {
    const double di = dr[i] / ms;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
      m[i * ld + j] += di * dc[j];
  }
}

// out = sum_ij P_ij * C_ij (block partials, then one CTA)
template <class COST>
__global__ void dot_cost_kernel(const CostView cv, const double* P, int64_t ld, double* partial) {
  const COST cost(cv);
  const int64_t n = cv.n;
  double s = 0.0;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const typename COST::Row row = cost.row(i);
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) s += P[i * ld + j] * cost.eval1(row, j);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

struct PlanFn {
  const CostView& cv;
  double a;
  const double *b, *r, *L;
  double* P;
  int64_t ld;
  cudaStream_t st;
  template <class COST>
  int run() {
    dim3 grid((unsigned)std::min<int64_t>((cv.n + 255) / 256, 16), (unsigned)std::min<int64_t>(cv.n, 8192));
    plan_kernel<COST><<<grid, 256, 0, st>>>(cv, a, b, r, L, P, ld);
    return LEANOT_OK;
  }
};

struct DotFn {
  const CostView& cv;
  const double* P;
  int64_t ld;
  double* partial;
  int nb;
  cudaStream_t st;
  template <class COST>
  int run() {
    dot_cost_kernel<COST><<<nb, 256, 0, st>>>(cv, P, ld, partial);
    return LEANOT_OK;
  }
};

// Dense primal-dual reference step (pdxg_reference_step, dxg.py:494-521), one row per CTA:
//   z_ij = decay lp_ij - tau (C_ij + two_sup d_j),  out_ij = z_ij - LSE_j z_ij  (lse_rows, core.py:67-70)
// exact row max, libdevice exp / log (the reference's np.exp / np.log), fixed reduction order.
template <class COST>
__global__ void __launch_bounds__(256) pdxg_rows_kernel(const CostView cv, const double* lp, int64_t ld, double decay,
                                                        double tau, double two_sup, const double* d, double* out) {
  __shared__ double red[8];
  __shared__ double bc;
  const COST cost(cv);
  const int64_t n = cv.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const typename COST::Row row = cost.row(i);
    double mx = -INFINITY;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      // the reference's NumPy operation order, no FMA contraction
      const double z = __dsub_rn(__dmul_rn(decay, lp[i * ld + j]),
                                 __dmul_rn(tau, __dadd_rn(cost.eval1(row, j), __dmul_rn(two_sup, d[j]))));
      out[i * ld + j] = z;
      mx = fmax(mx, z);
    }
    mx = warp_max(mx);
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red[0];
      for (int w = 1; w < 8; ++w) t = fmax(t, red[w]);
      bc = t;
    }
    __syncthreads();
    const double m = bc;
    double s = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) s += exp(out[i * ld + j] - m);
    s = warp_sum(s);
    __syncthreads();
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red[0];
      for (int w = 1; w < 8; ++w) t += red[w];
      bc = m + log(t);
    }
    __syncthreads();
    const double L = bc;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) out[i * ld + j] -= L;
    __syncthreads();
  }
}

// col_j = sum_i r_i exp(M_ij) in ascending row order (r @ np.exp(M), dxg.py:506, :512)
__global__ void pdxg_colsum_kernel(const double* M, int64_t n, int64_t ld, const double* r, double* col) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s = fma(r[i], exp(M[i * ld + j]), s);
    col[j] = s;
  }
}

struct PdxgRowsFn {
  const CostView& cv;
  const double* lp;
  int64_t ld;
  double decay, tau, two_sup;
  const double* d;
  double* out;
  cudaStream_t st;
  template <class COST>
  int run() {
    const int grid = (int)std::min<int64_t>(cv.n, 8192);
    pdxg_rows_kernel<COST><<<grid, 256, 0, st>>>(cv, lp, ld, decay, tau, two_sup, d, out);
    return LEANOT_OK;
  }
};

}  // namespace leanot

extern "C" {

// P = D_r p for weights (a, b): P_ij = r_i softmax_j(-(a C_ij + b_j)); L = row log-normalizers (leanot_row_lse)
int leanot_materialize_plan(const leanot_cost_t* cost, double a, const double* b, const double* r, const double* L,
                            double* P, int64_t ld, void* stream) {
  LEANOT_TRY(validate_cost(cost));
  LEANOT_TRY(ensure_init());
  if (ld < cost->n) { set_error("ld < n"); return LEANOT_EINVAL; }
  const CostView cv = make_view(*cost);
  PlanFn f{cv, a, b, r, L, P, ld, S_(stream)};
  LEANOT_TRY(LEANOT_DISPATCH_COST(cv, f));
  return check_launch("materialize_plan");
}

// Alg. 1 Round in place; scratch >= 2n + 2 doubles
int leanot_round_polytope(double* m, int64_t n, int64_t ld, const double* r, const double* c, double* scratch,
                          void* stream) {
  LEANOT_TRY(ensure_init());
  if (n < 1 || ld < n) { set_error("bad dense matrix"); return LEANOT_EINVAL; }
  cudaStream_t st = S_(stream);
  const int rb = (int)std::min<int64_t>((n + 7) / 8, 4096);
  const int cb = (int)std::min<int64_t>((n + 127) / 128, 4096);
  round_rows_kernel<<<rb, 256, 0, st>>>(m, n, ld, r);
  round_cols_kernel<<<cb, 128, 0, st>>>(m, n, ld, c);
  double* dr = scratch;
  double* dc = scratch + n;
  double* mass = scratch + 2 * n;
  round_deficit_rows_kernel<<<rb, 256, 0, st>>>(m, n, ld, r, dr);
  round_deficit_cols_kernel<<<cb, 128, 0, st>>>(m, n, ld, c, dc);
  sum_kernel<<<1, 1024, 0, st>>>(dr, n, mass);
  dim3 g((unsigned)std::min<int64_t>((n + 255) / 256, 16), (unsigned)std::min<int64_t>(n, 8192));
  round_outer_kernel<<<g, 256, 0, st>>>(m, n, ld, dr, dc, mass);
  return check_launch("round_polytope");
}

// out[0] = sum_ij P_ij C_ij; scratch >= 1024 doubles
int leanot_plan_cost(const leanot_cost_t* cost, const double* P, int64_t ld, double* out, double* scratch,
                     void* stream) {
  LEANOT_TRY(validate_cost(cost));
  LEANOT_TRY(ensure_init());
  const CostView cv = make_view(*cost);
  const int nb = (int)std::min<int64_t>(cost->n, 1024);
  DotFn f{cv, P, ld, scratch, nb, S_(stream)};
  LEANOT_TRY(LEANOT_DISPATCH_COST(cv, f));
  sum_kernel<<<1, 1024, 0, S_(stream)>>>(scratch, nb, out);
  return check_launch("plan_cost");
}

// pdxg_reference_step's row update (dxg.py:508-509, :514-515): out = z - lse_rows(z),
// z = decay lp - tau (C + two_sup d[None, :]); out may not alias lp
int leanot_pdxg_rows(const leanot_cost_t* cost, const double* lp, int64_t ld, double decay, double tau, double two_sup,
                     const double* d, double* out, void* stream) {
  LEANOT_TRY(validate_cost(cost));
  LEANOT_TRY(ensure_init());
  if (ld < cost->n) { set_error("ld < n"); return LEANOT_EINVAL; }
  if (lp == out) { set_error("pdxg_rows: out must not alias lp"); return LEANOT_EINVAL; }
  const CostView cv = make_view(*cost);
  PdxgRowsFn f{cv, lp, ld, decay, tau, two_sup, d, out, S_(stream)};
  LEANOT_TRY(LEANOT_DISPATCH_COST(cv, f));
  return check_launch("pdxg_rows");
}

// col = r @ exp(M) (dxg.py:505-506, :511-512)
int leanot_pdxg_colsum(const double* M, int64_t n, int64_t ld, const double* r, double* col, void* stream) {
  LEANOT_TRY(ensure_init());
  if (n < 1 || ld < n) { set_error("bad dense matrix"); return LEANOT_EINVAL; }
  const int grid = (int)std::min<int64_t>((n + 127) / 128, 4096);
  pdxg_colsum_kernel<<<grid, 128, 0, S_(stream)>>>(M, n, ld, r, col);
  return check_launch("pdxg_colsum");
}


}  // extern "C"
