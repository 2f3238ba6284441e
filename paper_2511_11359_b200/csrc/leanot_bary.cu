// DXG for entropic barycenters (Alg. 4; barycenter.py:108-151, 214-224).
//
// m marginals share the scalars a, s, t.  Both half-steps' weight sets of every
// marginal, {(a, b_k), (a_next, b_bar_k)}, depend only on the current state, so one
// sweep per marginal (pass A over both sets) yields all 2m row log-normalizers;
// the implicit barycenters r_now / r_bar follow from the sorted k-sum r-map
// (barycenter.py:90-97), and one column pass per marginal then produces both
// column marginals with row weights r_now / r_bar.  O(n) updates are the DXG ones
// per marginal, with the shared scalars advanced once.
// Included by leanot_lib.cu (single translation unit).

namespace leanot {

// coef[k][w][i][0..3] = (r_w[i] / S[k][w][i]) * EC{0..3}
__global__ void bary_coef_kernel(const double* S, const double* r, int m, int64_t nr, int64_t row0, int64_t n,
                                 double* coef) {
  const int64_t total = (int64_t)m * 2 * nr;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t li = t % nr;
    const int w = (int)((t / nr) % 2);
    const double g = r[w * n + row0 + li] / S[t];
    double* cf = coef + t * 4;
    cf[0] = g * EC0; cf[1] = g * EC1; cf[2] = g * EC2; cf[3] = g * EC3;
  }
}

// L[w][k][i] = m*LSTEP + log S[k][w][i]   (row log-normalizers, barycenter.py:78-87)
__global__ void bary_lse_kernel(const int64_t* mu, const double* S, int m, int64_t nr, double* L) {
  const int64_t total = (int64_t)m * 2 * nr;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t li = t % nr;
    const int w = (int)((t / nr) % 2);
    const int k = (int)(t / (2 * nr));
    L[((int64_t)w * m + k) * nr + li] = (double)mu[t] * LSTEP + log(S[t]);
  }
}

// dual of the penalized barycenter problem (barycenter.py:172-195): g_i = sum_k w_k log_z[k][i]
// (plain k order), out = LSE_i g_i
__global__ void bary_dual_reduce_kernel(const double* logz, const double* w, int m, int64_t n, double* out) {
  __shared__ double red[32];
  __shared__ double bc;
  double mx = -INFINITY;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double g = 0.0;
    for (int k = 0; k < m; ++k) g += w[k] * logz[k * n + i];
    mx = fmax(mx, g);
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = red[0];
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) t = fmax(t, red[q]);
    bc = t;
  }
  __syncthreads();
  const double gm = bc;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double g = 0.0;
    for (int k = 0; k < m; ++k) g += w[k] * logz[k * n + i];
    s += exp(g - gm);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) out[0] = gm + log(s);
}

// separable grid path (leanot_sep.cu)
static bool use_sep_bary(const leanot_bary_plan_t& P);
static int sep_bary_rows(const leanot_bary_plan_t& P, bool eval, cudaStream_t st);
static int sep_bary_cols(const leanot_bary_plan_t& P, cudaStream_t st);
static int sep_bary_eval(const leanot_bary_plan_t& P, cudaStream_t st);

static int validate_bary(const leanot_bary_plan_t* P) {
  if (!P) { set_error("null plan"); return LEANOT_EINVAL; }
  LEANOT_TRY(validate_cost(&P->cost));
  if (P->n != P->cost.n || P->row0 < 0 || P->row1 > P->n || P->row0 >= P->row1 || P->ns < P->n || (P->ns & 1) ||
      P->m < 1 || P->m > LEANOT_MAX_K || P->splits < 1 || P->nblk_upd < 1 || P->nblk_upd > 1024) {
    set_error("inconsistent barycenter plan (rows 0 <= row0 < row1 <= n; 1 <= m <= 16)");
    return LEANOT_EINVAL;
  }
  if (!(P->prm.eta > 0)) { set_error("barycenter solver requires eta > 0"); return LEANOT_EINVAL; }
  return LEANOT_OK;
}

static UpdArgs bary_upd(const leanot_bary_plan_t& P, int k) {
  UpdArgs U;
  const int64_t n = P.n;
  const int64_t ns = P.ns;
  U.n = n; U.col = P.col + (int64_t)k * 2 * n; U.c = P.c + k * ns; U.ct = P.c_tilde + k * ns;
  U.delta = P.delta + k * ns; U.b = P.b + k * ns; U.bprime = P.bprime + k * ns;
  U.b_bar = P.b_bar + k * ns; U.sd = P.sd + k * ns; U.partial = P.partial; U.scal = P.scal;
  const leanot_params_t& q = P.prm;
  const double sup = P.cost.sup_norm;
  U.A = 1.0 - q.tau_mu * q.eta_mu;
  U.B = 4.0 * q.tau_mu * sup;
  U.beta = q.beta;
  U.decay = 1.0 - q.tau_p * q.eta;
  U.G = 2.0 * q.tau_p * sup;
  U.twosup = 2.0 * sup;
  U.tau_p = q.tau_p;
  U.tau_p_eta = q.tau_p * q.eta;
  U.nblk = P.nblk_upd;
  U.zs_col = 2 * n;
  U.zs_vec = ns;
  return U;
}

static RowPassArgs bary_rowpass(const leanot_bary_plan_t& P, int k) {
  RowPassArgs A;
  memset(&A, 0, sizeof(A));
  const int64_t n = P.n, nr = P.row1 - P.row0;
  A.cost = make_view(P.cost);
  A.i0 = P.row0; A.i1 = P.row1;
  A.a = P.scal;
  A.b[0] = P.b + k * P.ns; A.b[1] = P.b_bar + k * P.ns;
  A.shift = P.shift + (int64_t)k * nr; A.shift_kstride = 0;
  A.S = P.S + (int64_t)k * 2 * nr; A.m_used = P.mu + (int64_t)k * 2 * nr;
  A.rowstat = P.rowstat + (int64_t)k * 3 * nr; A.sd = P.sd + k * P.ns;
  A.rw = nullptr; A.coef = nullptr;
  A.shift_next = P.shift + (int64_t)k * nr; A.next_from_k = 1;
  A.flags = P.flags;
  return A;
}

// marginals k and k + 1 in one pass A: sets {0, 1} = marginal k (now, bar), {2, 3} = k + 1
static RowPassArgs bary_rowpass2(const leanot_bary_plan_t& P, int k) {
  RowPassArgs A = bary_rowpass(P, k);
  const int64_t nr = P.row1 - P.row0;
  A.a = P.scal + 4;                               // [a, a_bar, a, a_bar] (bary_a4_kernel)
  A.b[2] = P.b + (k + 1) * P.ns; A.b[3] = P.b_bar + (k + 1) * P.ns;
  A.shift_kstride = nr; A.shift_kgroup = 2;       // marginal k + set / 2
  A.next_group = 2;                               // sets 1, 3 -> next shifts of k, k + 1
  A.rowstat = nullptr;
  return A;
}

__global__ void bary_a4_kernel(double* scal) {
  if (threadIdx.x < 4) scal[4 + threadIdx.x] = scal[threadIdx.x & 1];
}

// LEANOT_BARY_BATCH=0: one marginal per pass (A/B measurements); read per call
static int bary_batch() {
  const char* e = getenv("LEANOT_BARY_BATCH");
  return (e && e[0] == '0') ? 1 : 2;
}

}  // namespace leanot

extern "C" {

int leanot_bary_prepare(const leanot_bary_plan_t* P, double a, double s, double t, int init_shift, void* stream) {
  LEANOT_TRY(validate_bary(P));
  LEANOT_TRY(ensure_init());
  cudaStream_t st = S_(stream);
  const int64_t nr = P->row1 - P->row0;
  cudaMemsetAsync(P->flags, 0, 8, st);
  for (int k = 0; k < P->m; ++k) {
    UpdArgs U = bary_upd(*P, k);
    dxg_prepare_kernel<<<P->nblk_upd, 256, 0, st>>>(U, a, s, t);
    dxg_update3<<<P->nblk_upd, 256, 0, st>>>(U);
    if (init_shift) {
      fill_i64_kernel<<<(int)std::min<int64_t>((nr + 255) / 256, 1024), 256, 0, st>>>(
          P->shift + (int64_t)k * nr, nr, llrint(log((double)P->n) * (1.0 / LSTEP)));
    } else {
      RowPassArgs A = bary_rowpass(*P, k);
      LEANOT_TRY(launch_rowmax(A, 2, P->mu + (int64_t)k * 2 * nr, st));
      max_i64_pair_kernel<<<(int)std::min<int64_t>((nr + 255) / 256, 1024), 256, 0, st>>>(
          P->mu + (int64_t)k * 2 * nr, P->mu + (int64_t)k * 2 * nr + nr, P->shift + (int64_t)k * nr, nr);
    }
  }
  return check_launch("bary_prepare");
}

int leanot_bary_sweep(const leanot_bary_plan_t* P, int flags, void* stream) {
  LEANOT_TRY(validate_bary(P));
  LEANOT_TRY(ensure_init());
  cudaStream_t st = S_(stream);
  const int64_t n = P->n, nr = P->row1 - P->row0;
  const int m = P->m;
  if (nr != n) {
    set_error("row-sharded barycenter plans sweep through leanot_bary_rows / _rnorm / _cols");
    return LEANOT_EINVAL;
  }
  if (use_sep_bary(*P)) {
    // grid cost: separable O(n^1.5) row normalizers, r-maps, separable column sums
    LEANOT_TRY(sep_bary_rows(*P, (flags & LEANOT_SWEEP_EVAL) != 0, st));
    for (int w = 0; w < 2; ++w)
      launch_rmap(P->L + (int64_t)w * m * nr, m, n, P->w, P->scratch, P->partial, P->r + (int64_t)w * n, st);
    LEANOT_TRY(sep_bary_cols(*P, st));
    return check_launch("bary_sweep(separable)");
  }
  // plain sweeps: two marginals per launch (K = 4 weight sets {b_k, b_bar_k, b_k+1, b_bar_k+1}
  // share each read of C; a, a_bar mirrored into scal[4..7]); evaluation sweeps: one per marginal
  const bool eval = (flags & LEANOT_SWEEP_EVAL) != 0;
  const int kb = eval ? 1 : bary_batch();
  if (kb == 2) bary_a4_kernel<<<1, 32, 0, st>>>(P->scal);
  for (int k = 0; k < m; k += kb) {
    if (kb == 2 && k + 1 < m) {
      RowPassArgs A = bary_rowpass2(*P, k);
      LEANOT_TRY(launch_rowpass(A, 4, false, st));
    } else {
      RowPassArgs A = bary_rowpass(*P, k);
      LEANOT_TRY(launch_rowpass(A, 2, eval, st));
    }
  }
  const int64_t tot = (int64_t)m * 2 * nr;
  const int g = (int)std::min<int64_t>((tot + 255) / 256, 4096);
  bary_lse_kernel<<<g, 256, 0, st>>>(P->mu, P->S, m, nr, P->L);
  // r_now from the current weights, r_bar from the midpoint weights (barycenter.py:126, 137)
  for (int w = 0; w < 2; ++w)
    launch_rmap(P->L + (int64_t)w * m * nr, m, n, P->w, P->scratch, P->partial, P->r + (int64_t)w * n, st);
  bary_coef_kernel<<<g, 256, 0, st>>>(P->S, P->r, m, nr, P->row0, n, P->coef);
  // column sums: two marginals per launch as well (the per-set m / coef / col blocks of
  // marginals k and k + 1 are contiguous, so K = 4 indexes straight through them).  The
  // [a, a_bar, a, a_bar] copy is refreshed here too: evaluation sweeps skip the pass-A one.
  const int cb = bary_batch();
  if (cb == 2) bary_a4_kernel<<<1, 32, 0, st>>>(P->scal);
  for (int k = 0; k < m; k += cb) {
    const int K = cb == 2 && k + 1 < m ? 4 : 2;
    ColPassArgs B;
    memset(&B, 0, sizeof(B));
    B.cost = make_view(P->cost); B.i0 = P->row0; B.i1 = P->row1; B.a = K == 4 ? P->scal + 4 : P->scal;
    B.b[0] = P->b + k * P->ns; B.b[1] = P->b_bar + k * P->ns;
    if (K == 4) { B.b[2] = P->b + (k + 1) * P->ns; B.b[3] = P->b_bar + (k + 1) * P->ns; }
    B.m = P->mu + (int64_t)k * 2 * nr; B.coef = P->coef + (int64_t)k * 2 * nr * 4; B.slab = P->slab;
    B.splits = P->splits;
    LEANOT_TRY(launch_colpass(B, K, st));
    LEANOT_TRY(launch_slab_reduce(P->slab, P->splits, K, n, P->col + (int64_t)k * 2 * n, st));
  }
  return check_launch("bary_sweep");
}

int leanot_bary_update(const leanot_bary_plan_t* P, void* stream) {
  LEANOT_TRY(validate_bary(P));
  LEANOT_TRY(ensure_init());
  cudaStream_t st = S_(stream);
  // all m marginals in one launch per step (blockIdx.y = k); the shared scalars advance once
  const UpdArgs U = bary_upd(*P, 0);
  const dim3 g(P->nblk_upd, P->m);
  dxg_update1<<<g, 256, 0, st>>>(U);
  dxg_update2<<<g, 256, 0, st>>>(U, 1);
  dxg_update3<<<g, 256, 0, st>>>(U);
  return check_launch("bary_update");
}

// evalbuf layout: [k*4 + 0] cost_k, [k*4+1] sum_i r_i H(p_ki), [k*4+3] infeas_k; [64 + k*2] infeas_k, c.d_k;
// [127] LSE_i of the dual's g (barycenter.py:193-195)
int leanot_bary_eval(const leanot_bary_plan_t* P, void* stream) {
  LEANOT_TRY(validate_bary(P));
  LEANOT_TRY(ensure_init());
  cudaStream_t st = S_(stream);
  if (use_sep_bary(*P)) {
    LEANOT_TRY(sep_bary_eval(*P, st));
    return check_launch("bary_eval(separable)");
  }
  const int64_t n = P->n, nr = P->row1 - P->row0;
  const int m = P->m;
  for (int k = 0; k < m; ++k) {
    rowstats_reduce_kernel<<<1, 1024, 0, st>>>(nr, P->row0, P->r, P->S + (int64_t)k * 2 * nr,
                                               P->mu + (int64_t)k * 2 * nr, P->rowstat + (int64_t)k * 3 * nr, nullptr,
                                               P->evalbuf + k * 4);
    colstats_reduce_kernel<<<1, 1024, 0, st>>>(n, P->col + (int64_t)k * 2 * n, P->c + k * P->ns,
                                               P->delta + k * P->ns, P->evalbuf + 64 + k * 2);
    // log_z[k][i] = LSE_j(-(C_ij + 2 sup d_kj)/eta) (barycenter.py:186-191) into L (free after the sweep);
    // exact shift from the evaluation sweep's row minima min_j(C_ij + sd_kj) (one read of C)
    LEANOT_TRY(launch_rowlse(make_view(P->cost), P->row0, P->row1, P->sd + k * P->ns, 1.0, -1.0 / P->prm.eta,
                             P->L + (int64_t)k * nr, st, P->rowstat + (int64_t)k * 3 * nr + 2 * nr));
  }
  // LSE over this plan's rows (all rows single-process; a shard's rows otherwise, combined by the caller)
  bary_dual_reduce_kernel<<<1, 1024, 0, st>>>(P->L, P->w, m, nr, P->evalbuf + 127);
  return check_launch("bary_eval");
}

// ---- row-sharded sweep (multi-GPU): three phases around the caller's collectives ----

int leanot_bary_rows(const leanot_bary_plan_t* P, int flags, double* gmax, void* stream) {
  LEANOT_TRY(validate_bary(P));
  LEANOT_TRY(ensure_init());
  if (!gmax) { set_error("bary_rows: null gmax"); return LEANOT_EINVAL; }
  cudaStream_t st = S_(stream);
  const int64_t n = P->n, nr = P->row1 - P->row0;
  const int m = P->m;
  // plain sweeps: two marginals per launch (K = 4 weight sets {b_k, b_bar_k, b_k+1, b_bar_k+1}
  // share each read of C; a, a_bar mirrored into scal[4..7]); evaluation sweeps: one per marginal
  const bool eval = (flags & LEANOT_SWEEP_EVAL) != 0;
  const int kb = eval ? 1 : bary_batch();
  if (kb == 2) bary_a4_kernel<<<1, 32, 0, st>>>(P->scal);
  for (int k = 0; k < m; k += kb) {
    if (kb == 2 && k + 1 < m) {
      RowPassArgs A = bary_rowpass2(*P, k);
      LEANOT_TRY(launch_rowpass(A, 4, false, st));
    } else {
      RowPassArgs A = bary_rowpass(*P, k);
      LEANOT_TRY(launch_rowpass(A, 2, eval, st));
    }
  }
  const int64_t tot = (int64_t)m * 2 * nr;
  const int g = (int)std::min<int64_t>((tot + 255) / 256, 4096);
  bary_lse_kernel<<<g, 256, 0, st>>>(P->mu, P->S, m, nr, P->L);
  // g_w,i (sorted k-sum, barycenter.py:90-97) into r[w][row0 + i]; local maxima -> gmax[w]
  const int nblk = (int)std::min<int64_t>((nr + 255) / 256, 1024);
  for (int w = 0; w < 2; ++w) {
    bary_g_kernel<<<nblk, 256, 0, st>>>(P->L + (int64_t)w * m * nr, m, nr, P->w, P->r + (int64_t)w * n + P->row0,
                                        P->partial);
    reduce_max_kernel<<<1, 1024, 0, st>>>(P->partial, nblk, gmax + w);
  }
  return check_launch("bary_rows");
}

int leanot_bary_rnorm(const leanot_bary_plan_t* P, const double* gmax, double* esum, void* stream) {
  LEANOT_TRY(validate_bary(P));
  LEANOT_TRY(ensure_init());
  if (!gmax || !esum) { set_error("bary_rnorm: null scalars"); return LEANOT_EINVAL; }
  cudaStream_t st = S_(stream);
  const int64_t n = P->n, nr = P->row1 - P->row0;
  const int nblk = (int)std::min<int64_t>((nr + 255) / 256, 1024);
  for (int w = 0; w < 2; ++w) {
    double* rw = P->r + (int64_t)w * n + P->row0;
    // e_i = exp(g_i - global max), block partial sums, then their fixed-order total
    bary_e_kernel<<<nblk, 256, 0, st>>>(rw, nr, gmax + w, 1, rw, P->partial);
    sum_fixed_kernel<<<1, 1024, 0, st>>>(P->partial, nblk, esum + w);
  }
  return check_launch("bary_rnorm");
}

int leanot_bary_cols(const leanot_bary_plan_t* P, const double* esum, void* stream) {
  LEANOT_TRY(validate_bary(P));
  LEANOT_TRY(ensure_init());
  if (!esum) { set_error("bary_cols: null esum"); return LEANOT_EINVAL; }
  cudaStream_t st = S_(stream);
  const int64_t n = P->n, nr = P->row1 - P->row0;
  const int m = P->m;
  const int nblk = (int)std::min<int64_t>((nr + 255) / 256, 1024);
  for (int w = 0; w < 2; ++w) bary_norm_kernel<<<nblk, 256, 0, st>>>(P->r + (int64_t)w * n + P->row0, nr, esum + w, 1);
  const int64_t tot = (int64_t)m * 2 * nr;
  const int g = (int)std::min<int64_t>((tot + 255) / 256, 4096);
  bary_coef_kernel<<<g, 256, 0, st>>>(P->S, P->r, m, nr, P->row0, n, P->coef);
  bary_a4_kernel<<<1, 32, 0, st>>>(P->scal);
  const int cb = bary_batch();
  for (int k = 0; k < m; k += cb) {   // two marginals per read of C (as leanot_bary_sweep)
    const int K = cb == 2 && k + 1 < m ? 4 : 2;
    ColPassArgs B;
    memset(&B, 0, sizeof(B));
    B.cost = make_view(P->cost); B.i0 = P->row0; B.i1 = P->row1; B.a = K == 4 ? P->scal + 4 : P->scal;
    B.b[0] = P->b + k * P->ns; B.b[1] = P->b_bar + k * P->ns;
    if (K == 4) { B.b[2] = P->b + (k + 1) * P->ns; B.b[3] = P->b_bar + (k + 1) * P->ns; }
    B.m = P->mu + (int64_t)k * 2 * nr; B.coef = P->coef + (int64_t)k * 2 * nr * 4; B.slab = P->slab;
    B.splits = P->splits;
    LEANOT_TRY(launch_colpass(B, K, st));
    LEANOT_TRY(launch_slab_reduce(P->slab, P->splits, K, n, P->col + (int64_t)k * 2 * n, st));
  }
  return check_launch("bary_cols");
}

}  // extern "C"
