// Separable fast path for GridKernel costs.
//
// C_ij = (f(|r_i - r_j|) + f(|c_i - c_j|)) / scale, f(d) = d^p, on an H x W grid with
// row-major cells (core.py:200-236).  Every n^2 reduction of the DXG iteration factors
// into two 1-D reductions along the grid axes, in the log domain:
//   L_i   = LSE_j(-(a C_ij + b_j))             = LSE_rj( g(|ri-rj|) + LSE_cj( g(|ci-cj|) - b_(rj,cj) ) )
//   col_j = sum_i r_i exp(-(a C_ij + b_j) - L_i) = exp(-b_j + LSE_ri( g + LSE_ci( g + log r_i - L_i )))
// with g(d) = -a f(d)/scale.  Each stage is an "LSE-convolution" along one axis
// (H*W outputs, each an exact max-shifted LSE over W or H terms): O(n (H + W)) = O(n^1.5)
// work instead of O(n^2) -- 316 x 316 grid: 6.3e7 instead of 1e10 terms per pass.
// Evaluation statistics factor the same way (cost and sum p*b via log-weighted tables,
// the eta = 0 dual via min-plus convolutions).  Included by leanot_lib.cu.

namespace leanot {

// Y[p][q] = LSE_{q'} (X[p][q'] + g[|q-q'|])  (axis 1)   or   LSE_{p'} (X[p'][q] + g[|p-p'|])  (axis 0)
// MIN mode: min instead of LSE.  One thread per output; two passes (exact max, then the
// max-shifted sum with the table exp of leanot_common.cuh, zero integer shift).
template <bool MIN>
__global__ void __launch_bounds__(256) sep_axis_kernel(const double* __restrict__ X, const double* __restrict__ g,
                                                       int H, int W, int axis, double* __restrict__ Y) {
  extern __shared__ __align__(16) char smem[];
  uint32_t tb = 0;
  if (!MIN) {
    load_table(reinterpret_cast<double*>(smem));
    __syncthreads();
    tb = lane_tab_addr(smem);
  }
  const int64_t total = (int64_t)H * W;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(o / W), q = (int)(o % W);
    const int len = axis ? W : H;
    const int pos = axis ? q : p;
    const double* base = axis ? X + (int64_t)p * W : X + q;
    const int64_t stride = axis ? 1 : W;
    double m = INFINITY * (MIN ? 1.0 : -1.0);
    for (int t = 0; t < len; ++t) {
      const double v = base[t * stride] + g[abs(pos - t)];
      m = MIN ? fmin(m, v) : fmax(m, v);
    }
    if (MIN || m == -INFINITY) {
      Y[o] = m;
      continue;
    }
    double s = 0.0;
#pragma unroll 4
    for (int t = 0; t < len; ++t) texp_acc(tb, fmax(base[t * stride] + g[abs(pos - t)] - m, -1000.0), 0u, s);
    Y[o] = m + log(s);
  }
}

// g[d] = -a f(d) * inv (mode 0);  g[d] + log(f(d) * inv) (mode 1, -inf at d = 0);  f(d) * inv (mode 2);
// -f(d) * inv / eta (mode 3).  a read from device memory (graph-replay safe).
__global__ void sep_table_kernel(const double* a_ptr, int p, double inv, double eta, int D, int mode, double* g) {
  const double a = a_ptr ? *a_ptr : 0.0;
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < D; d += gridDim.x * blockDim.x) {
    const double dd = (double)d;
    const double f = p == 1 ? dd : (p == 2 ? dd * dd : dd * dd * dd);
    const double base = -a * (f * inv);
    if (mode == 0) g[d] = base;
    else if (mode == 1) g[d] = d == 0 ? -INFINITY : base + log(f * inv);
    else if (mode == 2) g[d] = f * inv;
    else g[d] = -(f * inv) / eta;
  }
}

// elementwise helpers over n cells
__global__ void sep_neg_kernel(const double* b, int64_t n, double* out) {  // out = -b
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = -b[i];
}
__global__ void sep_logw_kernel(const double* r, const double* L, int64_t n, double* out) {  // log r - L
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = r[i] > 0 ? log(r[i]) - L[i] : -INFINITY;
}
__global__ void sep_col_kernel(const double* V, const double* b, int64_t n, double* col) {  // exp(V - b)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    col[i] = exp(V[i] - b[i]);
}
__global__ void sep_logabsb_kernel(const double* b, int64_t n, double* out) {  // log|b| - b (b <= 0 after recentering)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = b[i] != 0.0 ? log(fabs(b[i])) - b[i] : -INFINITY;
}
__global__ void sep_scale_kernel(const double* x, double s, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[i] * s;
}

// per-row evaluation terms from the separable stats:
//   cost_i = exp(Cr_i - L_i) + exp(Cc_i - L_i)            (sum_j p_ij C_ij)
//   ent_i  = L_i + a cost_i - sgn_b exp(B_i - L_i)          (-sum_j p_ij log p_ij; B = log sum e^x |b|, b <= 0)
//   out[0] = sum r_i cost_i, out[1] = sum_{r_i>0} r_i ent_i, out[2] = sum r_i v_i
__global__ void sep_rowstats_kernel(int64_t n, const double* r, const double* L, const double* Cr, const double* Cc,
                                    const double* Bl, const double* a_ptr, const double* v, double* out) {
  const double a = *a_ptr;
  double cst = 0.0, ent = 0.0, inner = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double ri = r[i];
    const double ci = exp(Cr[i] - L[i]) + exp(Cc[i] - L[i]);
    cst += ri * ci;
    if (ri > 0.0) ent += ri * (L[i] + a * ci - exp(Bl[i] - L[i]));
    inner += ri * v[i];
  }
  cst = block_sum(cst);
  ent = block_sum(ent);
  inner = block_sum(inner);
  if (threadIdx.x == 0) { out[0] = cst; out[1] = ent; out[2] = inner; }
}

struct SepCtx {
  int H, W, p;
  int64_t n;
  double inv;
  cudaStream_t st;
  int nb;
  void axis(const double* X, const double* g, int ax, double* Y, bool mn = false) const {
    if (mn) {
      sep_axis_kernel<true><<<nb, 256, 0, st>>>(X, g, H, W, ax, Y);
    } else {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(sep_axis_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TAB_BYTES);
        attr = true;
      }
      sep_axis_kernel<false><<<nb, 256, TAB_BYTES, st>>>(X, g, H, W, ax, Y);
    }
  }
  void table(const double* a_ptr, int mode, double* g, double eta = 1.0) const {
    const int D = H > W ? H : W;
    sep_table_kernel<<<(D + 255) / 256, 256, 0, st>>>(a_ptr, p, inv, eta, D, mode, g);
  }
  int eg() const { return (int)std::min<int64_t>((n + 255) / 256, 4096); }
};

static SepCtx make_sep(const leanot_cost_t& c, cudaStream_t st) {
  SepCtx s;
  s.H = c.height; s.W = c.width; s.p = c.p; s.n = c.n; s.inv = c.inv_scale; s.st = st;
  s.nb = (int)std::min<int64_t>((c.n + 255) / 256, (int64_t)num_sms() * 3);
  return s;
}

// scratch layout (doubles): 6 n-vectors + 4 tables of D
static int64_t sep_ws_doubles(const leanot_cost_t& c) {
  const int D = c.height > c.width ? c.height : c.width;
  return 6 * c.n + 4 * (int64_t)D + 64;
}

static bool sep_enabled_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LEANOT_GRID_SEPARABLE");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// DXG sweep on a grid cost, both weight sets, single process: writes col (2n), L into S-slots
// (S = 1, m = 0 so that downstream code sees L_i = log S + m*LSTEP is not used), and eval stats.
static int sep_dxg_sweep(const leanot_dxg_plan_t& P, bool eval, cudaStream_t st) {
  const SepCtx s = make_sep(P.cost, st);
  const int64_t n = P.n;
  const int D = s.H > s.W ? s.H : s.W;
  double* ws = P.slab;  // engine sizes the slab >= sep_ws_doubles for grid costs
  double *T = ws, *L = ws + n, *U = ws + 2 * n, *V = ws + 3 * n, *X = ws + 4 * n, *Y = ws + 5 * n;
  double *g = ws + 6 * n, *g2 = g + D, *g3 = g2 + D, *g4 = g3 + D;
  const int eg = s.eg();
  for (int k = 0; k < 2; ++k) {
    const double* bk = k == 0 ? P.b : P.b_bar;
    s.table(P.scal + k, 0, g);
    sep_neg_kernel<<<eg, 256, 0, st>>>(bk, n, X);
    s.axis(X, g, 1, T);
    s.axis(T, g, 0, L);
    if (eval && k == 0) {
      // cost: log sum_j e^{x_ij} f(dr)/s  and  ... f(dc)/s
      s.table(P.scal, 1, g2);
      double* Cr = P.rowstat;           // nr
      double* Cc = P.rowstat + n;       // nr
      s.axis(T, g2, 0, Cr);             // f(dr) weight on the row stage
      s.axis(X, g2, 1, Y);              // f(dc) weight on the column stage
      s.axis(Y, g, 0, Cc);
      // B = log sum_j e^{x_ij} |b_j|
      sep_logabsb_kernel<<<eg, 256, 0, st>>>(bk, n, Y);
      s.axis(Y, g, 1, U);
      s.axis(U, g, 0, V);
      double* Bl = P.bprime;            // scratch n-vector free during the sweep
      cudaMemcpyAsync(Bl, V, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
      // dual row reductions of C + sd (min-plus for eta = 0, LSE of -(C + sd)/eta otherwise)
      double* dv = P.rowstat + 2 * n;
      if (P.prm.eta > 0) {
        s.table(nullptr, 3, g3, P.prm.eta);
        sep_scale_kernel<<<eg, 256, 0, st>>>(P.sd, -1.0 / P.prm.eta, n, Y);
        s.axis(Y, g3, 1, U);
        s.axis(U, g3, 0, dv);
      } else {
        s.table(nullptr, 2, g4);
        s.axis(P.sd, g4, 1, U, true);
        s.axis(U, g4, 0, dv, true);
      }
      // keep L of weight set 0 for the reduce
      cudaMemcpyAsync(P.S, L, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
    }
    // column marginal with row weights r
    sep_logw_kernel<<<eg, 256, 0, st>>>(P.r, L, n, X);
    s.axis(X, g, 1, U);
    s.axis(U, g, 0, V);
    sep_col_kernel<<<eg, 256, 0, st>>>(V, bk, n, P.col + k * n);
  }
  return LEANOT_OK;
}

static int sep_dxg_eval(const leanot_dxg_plan_t& P, cudaStream_t st) {
  const int64_t n = P.n;
  sep_rowstats_kernel<<<1, 1024, 0, st>>>(n, P.r, P.S, P.rowstat, P.rowstat + n, P.bprime, P.scal,
                                          P.rowstat + 2 * n, P.evalbuf);
  colstats_reduce_kernel<<<1, 1024, 0, st>>>(n, P.col, P.c, P.delta, P.evalbuf + 3);
  return LEANOT_OK;
}

// ---- barycenter (leanot_bary.cu) on a grid cost -------------------------------------
static bool use_sep_bary(const leanot_bary_plan_t& P) {
  return P.cost.kind == LEANOT_COST_GRID && sep_enabled_env();
}

// all 2m row log-normalizers into P.L ([w][k][i]); eval: per-k stats of weight set 0
static int sep_bary_rows(const leanot_bary_plan_t& P, bool eval, cudaStream_t st) {
  const SepCtx s = make_sep(P.cost, st);
  const int64_t n = P.n, ns = P.ns;
  const int m = P.m;
  const int D = s.H > s.W ? s.H : s.W;
  double* ws = P.slab;
  double *T = ws, *U = ws + n, *V = ws + 2 * n, *X = ws + 3 * n, *Y = ws + 4 * n;
  double *g = ws + 6 * n, *g2 = g + D;
  const int eg = s.eg();
  for (int w = 0; w < 2; ++w) {
    s.table(P.scal + w, 0, g);
    if (eval && w == 0) s.table(P.scal, 1, g2);
    for (int k = 0; k < m; ++k) {
      const double* bk = (w == 0 ? P.b : P.b_bar) + k * ns;
      double* L = P.L + ((int64_t)w * m + k) * n;
      sep_neg_kernel<<<eg, 256, 0, st>>>(bk, n, X);
      s.axis(X, g, 1, T);
      s.axis(T, g, 0, L);
      if (eval && w == 0) {
        double* Cr = P.rowstat + (int64_t)k * 3 * n;
        double* Cc = Cr + n;
        s.axis(T, g2, 0, Cr);
        s.axis(X, g2, 1, Y);
        s.axis(Y, g, 0, Cc);
        sep_logabsb_kernel<<<eg, 256, 0, st>>>(bk, n, Y);
        s.axis(Y, g, 1, U);
        s.axis(U, g, 0, P.S + (int64_t)k * 2 * n + n);   // B_k (log sum e^x |b|)
        cudaMemcpyAsync(P.S + (int64_t)k * 2 * n, L, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
      }
    }
  }
  (void)V;
  return LEANOT_OK;
}

// column marginals of all (k, w) with row weights r_w (P.r, after the r-maps)
static int sep_bary_cols(const leanot_bary_plan_t& P, cudaStream_t st) {
  const SepCtx s = make_sep(P.cost, st);
  const int64_t n = P.n, ns = P.ns;
  const int m = P.m;
  const int D = s.H > s.W ? s.H : s.W;
  double* ws = P.slab;
  double *U = ws + n, *V = ws + 2 * n, *X = ws + 3 * n;
  double* g = ws + 6 * n;
  (void)D;
  const int eg = s.eg();
  for (int w = 0; w < 2; ++w) {
    s.table(P.scal + w, 0, g);
    for (int k = 0; k < m; ++k) {
      const double* bk = (w == 0 ? P.b : P.b_bar) + k * ns;
      sep_logw_kernel<<<eg, 256, 0, st>>>(P.r + w * n, P.L + ((int64_t)w * m + k) * n, n, X);
      s.axis(X, g, 1, U);
      s.axis(U, g, 0, V);
      sep_col_kernel<<<eg, 256, 0, st>>>(V, bk, n, P.col + (int64_t)k * 2 * n + w * n);
    }
  }
  return LEANOT_OK;
}

static int sep_bary_eval(const leanot_bary_plan_t& P, cudaStream_t st) {
  const SepCtx s = make_sep(P.cost, st);
  const int64_t n = P.n, ns = P.ns;
  const int m = P.m;
  const int D = s.H > s.W ? s.H : s.W;
  double* ws = P.slab;
  double *U = ws + n, *Y = ws + 4 * n, *zero = ws + 5 * n;
  double* g3 = ws + 6 * n + 2 * D;
  const int eg = s.eg();
  cudaMemsetAsync(zero, 0, n * sizeof(double), st);
  s.table(nullptr, 3, g3, P.prm.eta);
  for (int k = 0; k < m; ++k) {
    const double* Cr = P.rowstat + (int64_t)k * 3 * n;
    sep_rowstats_kernel<<<1, 1024, 0, st>>>(n, P.r, P.S + (int64_t)k * 2 * n, Cr, Cr + n,
                                            P.S + (int64_t)k * 2 * n + n, P.scal, zero, P.evalbuf + k * 4);
    colstats_reduce_kernel<<<1, 1024, 0, st>>>(n, P.col + (int64_t)k * 2 * n, P.c + k * ns, P.delta + k * ns,
                                               P.evalbuf + 64 + k * 2);
    // log_z[k] = LSE_j(-(C_ij + sd_kj)/eta) (barycenter.py:186-191)
    sep_scale_kernel<<<eg, 256, 0, st>>>(P.sd + k * ns, -1.0 / P.prm.eta, n, Y);
    s.axis(Y, g3, 1, U);
    s.axis(U, g3, 0, P.L + (int64_t)k * n);
  }
  bary_dual_reduce_kernel<<<1, 1024, 0, st>>>(P.L, P.w, m, n, P.evalbuf + 127);
  return LEANOT_OK;
}

static bool use_sep(const leanot_dxg_plan_t& P) {
  return P.cost.kind == LEANOT_COST_GRID && P.row0 == 0 && P.row1 == P.n && sep_enabled_env();
}

}  // namespace leanot

extern "C" {

int64_t leanot_grid_sep_ws_doubles(const leanot_cost_t* cost) { return leanot::sep_ws_doubles(*cost); }

// standalone separable primitives (tests / barycenter): L = row LSE of -(a C + b), col = sum_i r_i softmax
int leanot_grid_sep_lse(const leanot_cost_t* cost, const double* a_dev, const double* b, double* L, double* ws,
                        void* stream) {
  using namespace leanot;
  LEANOT_TRY(validate_cost(cost));
  if (cost->kind != LEANOT_COST_GRID) { set_error("separable path needs a grid cost"); return LEANOT_EINVAL; }
  LEANOT_TRY(ensure_init());
  cudaStream_t st = S_(stream);
  const SepCtx s = make_sep(*cost, st);
  const int64_t n = cost->n;
  double *T = ws, *X = ws + n, *g = ws + 2 * n;
  s.table(a_dev, 0, g);
  sep_neg_kernel<<<s.eg(), 256, 0, st>>>(b, n, X);
  s.axis(X, g, 1, T);
  s.axis(T, g, 0, L);
  return check_launch("grid_sep_lse");
}

int leanot_grid_sep_colsum(const leanot_cost_t* cost, const double* a_dev, const double* b, const double* logw,
                           double* col, double* ws, void* stream) {
  using namespace leanot;
  LEANOT_TRY(validate_cost(cost));
  if (cost->kind != LEANOT_COST_GRID) { set_error("separable path needs a grid cost"); return LEANOT_EINVAL; }
  LEANOT_TRY(ensure_init());
  cudaStream_t st = S_(stream);
  const SepCtx s = make_sep(*cost, st);
  const int64_t n = cost->n;
  double *U = ws, *V = ws + n, *g = ws + 2 * n;
  s.table(a_dev, 0, g);
  s.axis(logw, g, 1, U);
  s.axis(U, g, 0, V);
  sep_col_kernel<<<s.eg(), 256, 0, st>>>(V, b, n, col);
  return check_launch("grid_sep_colsum");
}

}  // extern "C"
