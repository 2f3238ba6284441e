// Log-domain Sinkhorn and IBP baselines on the DXG sweep machinery (sinkhorn.py:47-228;
// SURVEY.md §8f item 1).  Row LSEs reuse rowlse_kernel; the column LSE
//   L_j = LSE_i((phi_i - C_ij)/eta)                       (sinkhorn.py:47-62)
// is one streaming pass with a running max per (column, row split), merged across
// splits in fixed order (the reference merges its 128-row blocks the same way).
// Included by leanot_lib.cu (single translation unit).

namespace leanot {

constexpr int CL_THREADS = 256;
constexpr int CL_V = 4;
constexpr int CL_TILE = CL_THREADS * CL_V;

// online (max, sum) for one value z: s*exp(m - z) + 1 when z raises the max
__device__ __forceinline__ void online_add(uint32_t tb, double z, double& m, double& s) {
  if (z > m) {
    s = (m == -INFINITY) ? 0.0 : s * texp(tb, fmax(m - z, -1000.0), 0u);
    m = z;
  }
  texp_acc(tb, fmax(z - m, -1000.0), 0u, s);
}

template <class COST>
__global__ void __launch_bounds__(CL_THREADS) collse_kernel(const CostView cv, int64_t i0, int64_t i1, const double* pre,
                                                          double inv, int splits, double* slab_m, double* slab_s) {
  extern __shared__ __align__(16) char smem[];
  load_table(reinterpret_cast<double*>(smem));
  __syncthreads();
  const uint32_t tb = lane_tab_addr(smem);
  const COST cost(cv);
  const int64_t n = cv.n, nr = i1 - i0;
  const int64_t ntiles = (n + CL_TILE - 1) / CL_TILE;
  const int64_t rps = (nr + splits - 1) / splits;
  for (int64_t it = blockIdx.x; it < ntiles * splits; it += gridDim.x) {
    const int64_t tile = it % ntiles, split = it / ntiles;
    const int64_t j = tile * CL_TILE + CL_V * threadIdx.x;
    const int nv = (int)(n - j < 0 ? 0 : (n - j > CL_V ? CL_V : n - j));
    double m[CL_V], s[CL_V];
#pragma unroll
    for (int v = 0; v < CL_V; ++v) { m[v] = -INFINITY; s[v] = 0.0; }
    const int64_t r0 = i0 + split * rps, r1 = i1 < r0 + rps ? i1 : r0 + rps;
    if (nv > 0) {
      for (int64_t i = r0; i < r1; ++i) {
        const typename COST::Row row = cost.row(i);
        const double p = __ldg(pre + (i - i0));
#pragma unroll
        for (int v = 0; v < CL_V; ++v)
          if (v < nv) online_add(tb, fma(cost.eval1(row, j + v), -inv, p), m[v], s[v]);
      }
    }
#pragma unroll
    for (int v = 0; v < CL_V; ++v)
      if (v < nv) {
        slab_m[split * n + j + v] = m[v];
        slab_s[split * n + j + v] = s[v];
      }
  }
}

// L_j = M + log(sum_s s_s exp(m_s - M)) over splits in fixed order
__global__ void collse_merge_kernel(const double* slab_m, const double* slab_s, int splits, int64_t n, double* L) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double M = -INFINITY;
    for (int q = 0; q < splits; ++q) M = fmax(M, slab_m[q * n + j]);
    double S = 0.0;
    for (int q = 0; q < splits; ++q) {
      const double mq = slab_m[q * n + j];
      if (mq > -INFINITY) S += slab_s[q * n + j] * exp(mq - M);
    }
    L[j] = M + log(S);
  }
}

__global__ void scale_vec_kernel(const double* x, double a, int64_t n, double* y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] * a;
}

// out = eta*log(w) - eta*L   (phi update, sinkhorn.py:98; also psi with c)
__global__ void eta_log_minus_kernel(const double* w, const double* L, double eta, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = eta * log(w[i]) - eta * L[i];
}

// psi_new = eta*log c - eta*L; gap = sum_j |c_j expm1((psi_j - psi_new_j)/eta)| (sinkhorn.py:99-102)
__global__ void sinkhorn_psi_kernel(const double* c, const double* L, const double* psi, double eta, int64_t n,
                                    double* psi_new, double* gap) {
  double g = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const double pn = eta * log(c[j]) - eta * L[j];
    psi_new[j] = pn;
    g += fabs(c[j] * expm1((psi[j] - pn) / eta));
  }
  g = block_sum(g);
  if (threadIdx.x == 0) *gap = g;
}

// <phi, r> + <psi, c> - eta * LSE_i(phi_i/eta + L_i)   (eot_dual_value, sinkhorn.py:120-136)
__global__ void eot_dual_kernel(const double* phi, const double* psi, const double* r, const double* c, const double* L,
                                double eta, int64_t n, double* out) {
  __shared__ double bc;
  double mx = -INFINITY;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, phi[i] / eta + L[i]);
  mx = warp_max(mx);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = red[0];
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) t = fmax(t, red[q]);
    bc = t;
  }
  __syncthreads();
  const double M = bc;
  double s = 0.0, pr = 0.0, pc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    s += exp(phi[i] / eta + L[i] - M);
    pr += phi[i] * r[i];
    pc += psi[i] * c[i];
  }
  s = block_sum(s);
  pr = block_sum(pr);
  pc = block_sum(pc);
  if (threadIdx.x == 0) out[0] = pr + pc - eta * (M + log(s));
}

// normalized column marginal of the Sinkhorn plan: col_j proportional to exp(psi_j/eta + L_j) (sinkhorn.py:139-150)
__global__ void sinkhorn_colmarg_kernel(const double* psi, const double* L, double eta, int64_t n, double* col) {
  __shared__ double bc;
  __shared__ double red[32];
  double mx = -INFINITY;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) mx = fmax(mx, psi[j] / eta + L[j]);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = red[0];
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) t = fmax(t, red[q]);
    bc = t;
  }
  __syncthreads();
  const double M = bc;
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const double e = exp(psi[j] / eta + L[j] - M);
    col[j] = e;
    s += e;
  }
  s = block_sum(s);
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) col[j] = col[j] / s;
}

// IBP row step (sinkhorn.py:222-224): log_r = sum_k w_k (phi_k/eta + RL_k) (k order);
// phi_k = eta*log_r - eta*RL_k
__global__ void ibp_row_kernel(const double* w, int m, int64_t n, double eta, const double* RL, double* phis,
                               double* log_r) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double lr = 0.0;
    for (int k = 0; k < m; ++k) lr += w[k] * (phis[k * n + i] / eta + RL[k * n + i]);
    log_r[i] = lr;
    for (int k = 0; k < m; ++k) phis[k * n + i] = eta * lr - eta * RL[k * n + i];
  }
}

struct ColLseFn {
  const CostView& cv;
  int64_t i0, i1;
  const double* pre;
  double inv;
  int splits;
  double *sm, *ss;
  cudaStream_t st;
  template <class COST>
  int run() {
    auto kern = collse_kernel<COST>;
    static bool attr = false;
    if (!attr) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TAB_BYTES) != cudaSuccess)
        return LEANOT_ECUDA;
      attr = true;
    }
    const int64_t items = ((cv.n + CL_TILE - 1) / CL_TILE) * splits;
    int grid = (int)std::min<int64_t>(items, (int64_t)num_sms() * 3);
    if (grid < 1) return LEANOT_OK;
    kern<<<grid, CL_THREADS, TAB_BYTES, st>>>(cv, i0, i1, pre, inv, splits, sm, ss);
    return LEANOT_OK;
  }
};

}  // namespace leanot

extern "C" {

int64_t leanot_col_lse_ws_doubles(int64_t n, int64_t rows) {
  int splits = 1;
  leanot_dxg_default_splits(n, rows, &splits);
  return rows + 2 * (int64_t)splits * n + 16;
}

// L_j = LSE_i((phi_i - C_ij)/eta) over rows [row0,row1) (sinkhorn.py:47-62)
int leanot_col_lse(const leanot_cost_t* cost, int64_t row0, int64_t row1, const double* phi, double eta, double* L,
                   double* ws, void* stream) {
  LEANOT_TRY(validate_cost(cost));
  LEANOT_TRY(ensure_init());
  if (!(eta > 0)) { set_error("col_lse needs eta > 0"); return LEANOT_EINVAL; }
  if (row0 < 0 || row1 > cost->n || row0 >= row1) { set_error("bad row range"); return LEANOT_EINVAL; }
  cudaStream_t st = S_(stream);
  const int64_t n = cost->n, nr = row1 - row0;
  int splits = 1;
  leanot_dxg_default_splits(n, nr, &splits);
  double* pre = ws;
  double* sm = ws + nr;
  double* ss = sm + (int64_t)splits * n;
  const double inv = 1.0 / eta;
  scale_vec_kernel<<<(int)std::min<int64_t>((nr + 255) / 256, 1024), 256, 0, st>>>(phi + row0, inv, nr, pre);
  const CostView cv = make_view(*cost);
  ColLseFn f{cv, row0, row1, pre, inv, splits, sm, ss, st};
  LEANOT_TRY(LEANOT_DISPATCH_COST(cv, f));
  collse_merge_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st>>>(sm, ss, splits, n, L);
  return check_launch("col_lse");
}

int leanot_eta_log_minus(const double* w, const double* L, double eta, int64_t n, double* out, void* stream) {
  LEANOT_TRY(ensure_init());
  eta_log_minus_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, S_(stream)>>>(w, L, eta, n, out);
  return check_launch("eta_log_minus");
}

int leanot_sinkhorn_psi(const double* c, const double* L, const double* psi, double eta, int64_t n, double* psi_new,
                        double* gap, void* stream) {
  LEANOT_TRY(ensure_init());
  sinkhorn_psi_kernel<<<1, 1024, 0, S_(stream)>>>(c, L, psi, eta, n, psi_new, gap);
  return check_launch("sinkhorn_psi");
}

int leanot_eot_dual(const double* phi, const double* psi, const double* r, const double* c, const double* L,
                    double eta, int64_t n, double* out, void* stream) {
  LEANOT_TRY(ensure_init());
  eot_dual_kernel<<<1, 1024, 0, S_(stream)>>>(phi, psi, r, c, L, eta, n, out);
  return check_launch("eot_dual");
}

int leanot_sinkhorn_colmarg(const double* psi, const double* L, double eta, int64_t n, double* col, void* stream) {
  LEANOT_TRY(ensure_init());
  sinkhorn_colmarg_kernel<<<1, 1024, 0, S_(stream)>>>(psi, L, eta, n, col);
  return check_launch("sinkhorn_colmarg");
}

int leanot_ibp_rows(const double* w, int m, int64_t n, double eta, const double* RL, double* phis, double* log_r,
                    void* stream) {
  LEANOT_TRY(ensure_init());
  ibp_row_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, S_(stream)>>>(w, m, n, eta, RL, phis,
                                                                                           log_r);
  return check_launch("ibp_rows");
}

}  // extern "C"
