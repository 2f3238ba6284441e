/*
 * leanot_b200.h -- C ABI of the B200-native DXG hot path (libleanot_b200.so).
 *
 * The reference (`leanot`, /root/reference/pkg/src/leanot) is pure Python/NumPy;
 * its only extension point on this path is the CostKernel plugin protocol
 * (core.py:167-192) consumed by the streamed sweeps of dxg.py / barycenter.py.
 * This library replaces those sweeps and the O(n) updates.  Every entry point:
 *   - takes raw DEVICE pointers + sizes (no torch types), plus a cudaStream_t
 *     (passed as void*; NULL = legacy default stream), and is stream-ordered;
 *   - never allocates persistent memory and never frees caller memory;
 *   - returns 0 on success, or a negative LEANOT_E* code with a message
 *     retrievable from leanot_last_error() (thread-local); no C++ exception
 *     crosses the boundary.  Invalid arguments are LEANOT_EINVAL, which the
 *     Python layer maps to ValueError exactly where the reference raises it.
 * All arithmetic is IEEE binary64.
 */
#ifndef LEANOT_B200_H
#define LEANOT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LEANOT_ABI_VERSION 2

#define LEANOT_OK 0
#define LEANOT_EINVAL (-1)
#define LEANOT_ECUDA (-2)
#define LEANOT_EINTERNAL (-3)

#define LEANOT_MAX_K 16

/* cost kinds: ExplicitKernel (core.py:239), ColorKernel (core.py:264), GridKernel (core.py:200) */
#define LEANOT_COST_STORED 0
#define LEANOT_COST_POINTS 1
#define LEANOT_COST_GRID 2

/* Device view of a CostKernel (core.py:167-192).  Normalized entries are
 * C_ij = mat[(i-row_base)*ld + j] (STORED, already divided by scale) or
 * raw_ij * inv_scale (POINTS: sum_d |f_id - f_jd|^p; GRID: |drow|^p + |dcol|^p). */
typedef struct leanot_cost {
  int32_t kind;
  int32_t p;          /* exponent 1..3 (POINTS / GRID) */
  int32_t dim;        /* POINTS feature dimension 1..4 */
  int32_t height;     /* GRID */
  int32_t width;      /* GRID */
  int32_t _pad;
  int64_t n;          /* number of columns (= global number of rows) */
  int64_t ld;         /* STORED row stride in doubles (>= n) */
  int64_t row_base;   /* STORED: global index of the first row held in mat */
  const double* mat;          /* STORED */
  const double* feat;         /* POINTS: n x dim row-major, 16-byte aligned */
  const double* grid_coords;  /* GRID: [row index (n) | column index (n)] as doubles */
  double inv_scale;   /* 1/scale for on-the-fly kinds */
  double sup_norm;    /* ||C||_inf after normalization: 1 or 0 */
  const double* norms;/* POINTS, p = 2, optional: leanot_points_norms output (|f_j - mu|^2, then the
                       * centered features).  When set, the non-evaluation DXG sweeps use the
                       * expanded form a C_ij = a inv (|g_i|^2 + |g_j|^2 - 2 g_i.g_j), g = f - mu,
                       * whose row constant cancels in the row softmax (dxg.py:199-202) */
} leanot_cost_t;

/* K weight sets {a_k, b_k}: rows softmax_j(-(a_k C_ij + b_kj)) (dxg.py:185-190).
 * a is a device array of K scalars so CUDA-graph replays see updated values. */
typedef struct leanot_wsets {
  int32_t K;
  int32_t _pad;
  const double* a;
  const double* b[LEANOT_MAX_K];
} leanot_wsets_t;

/* DxgParams (dxg.py:100-128) */
typedef struct leanot_params {
  double eta, eta_mu, tau_p, tau_mu, beta, alpha;
} leanot_params_t;

/* Solver workspace for dxg.solve / dxg_step (dxg.py:261-279, 420-472).  All
 * pointers are device memory allocated by the caller.  Rows [row0,row1) are
 * the rows this process sweeps (row sharding across GPUs); column vectors are
 * full length n.  Sizes: nr = row1-row0, K = 2. */
typedef struct leanot_dxg_plan {
  leanot_cost_t cost;
  leanot_params_t prm;
  int64_t n, row0, row1;
  int32_t splits;       /* row splits of the column pass (partial slabs) */
  int32_t nblk_upd;     /* number of CTAs of the O(n) update kernels */
  const double* r;      /* n  row marginal */
  const double* c;      /* n  column marginal */
  const double* c_tilde;/* n  c + alpha/n */
  double* delta;        /* n  LogOddsField.delta (state) */
  double* b;            /* n  TransportLogWeights.b (state) */
  double* b_bar;        /* n  midpoint weights (derived) */
  double* bprime;       /* n  scratch (pre-max b) */
  double* sd;           /* n  2*sup*tanh(delta/2) of the state (dual shift) */
  double* scal;         /* 8  device scalars: a, a_bar, s, t, sweep count, ... */
  int64_t* shift;       /* nr row shift (units of ln2/512) for the next sweep */
  int64_t* m;           /* 2*nr shifts used by the current sweep */
  double* S;            /* 2*nr row sums */
  double* coef;         /* 2*nr*4 column-pass polynomial coefficients */
  double* rowstat;      /* 3*nr  sum e*C, sum e*x, row min (evaluation sweeps) */
  double* slab;         /* splits*2*n column partials */
  double* col;          /* 2*n  reduced column marginals (col_now | col_bar) */
  double* partial;      /* 2*nblk_upd block maxima */
  double* evalbuf;      /* 16 evaluation scalars */
  int32_t* flags;       /* 2 + 4*nr int32: fixup list [count, -, (k, li) pairs]; up to 2 weight sets x nr rows */
  double* beta;         /* 2*((n+1)&~1) scratch for expanded-form sweeps (cost.norms set); may be null */
} leanot_dxg_plan_t;

/* ---- library ---------------------------------------------------------- */
int leanot_version(void);
const char* leanot_last_error(void);
int leanot_device_sm_count(int device, int* out);
/* column-pass row splits the engine sizes plan.slab with (splits*2*n doubles) for n columns, `rows` rows */
int leanot_dxg_default_splits(int64_t n, int64_t rows, int* out);

/* ---- cost kernels (core.py:167-288) ----------------------------------- */
/* rows [i0,i1) of the normalized cost into out (row-major, stride ldo): CostKernel.block */
int leanot_cost_block(const leanot_cost_t* cost, int64_t i0, int64_t i1, double* out, int64_t ldo, void* stream);
/* out[0] = max and out[1] = -min over all entries of the raw matrix (ExplicitKernel scale and the
   negative-entry check, core.py:252-258); scratch holds 2048 doubles */
int leanot_stored_max(const double* mat, int64_t rows, int64_t cols, int64_t ld, double* out, double* scratch, void* stream);
/* mat /= scale (in place, IEEE division as core.py:258) */
int leanot_stored_normalize(double* mat, int64_t rows, int64_t cols, int64_t ld, double scale, void* stream);
/* raw sup over all pairs of ||f_i - f_j||_p^p (ColorKernel scale, core.py:279-284) */
int leanot_points_sup(const double* feat, int64_t n, int dim, int p, double* out, double* scratch, void* stream);
/* leanot_cost_t.norms of a POINTS p = 2 cost: out = [|f_j - mu|^2 (n, padded to an even count np) |
 * f_j - mu (n x dim, row-major) | mu (dim)], mu = the per-dimension feature mean (fixed-order
 * reduction).  The expanded-form sweeps run on the centered features (translation-invariant cost,
 * smaller cancellation error); out holds np + n*dim + dim doubles. */
int leanot_points_norms(const double* feat, int64_t n, int dim, double* out, void* stream);
/* benchmark instance: C_ij = splitmix64(seed,i,j) -> U[0,1), C[0][n-1] = 1 (oracle/leanot_oracle.py:hash_u01) */
int leanot_hash_fill(double* mat, int64_t row0, int64_t rows, int64_t n, int64_t ld, uint64_t seed, void* stream);

/* ---- sweeps ------------------------------------------------------------ */
/* column_marginal for K weight sets (dxg.py:193-208): out[k*n + j] = sum_i r_i softmax_j.
 * Robust (computes row maxima first); workspace: ws of leanot_sweep_ws_doubles() doubles. */
int64_t leanot_sweep_ws_doubles(int64_t n, int64_t rows, int K);
int leanot_column_marginals(const leanot_cost_t* cost, int64_t row0, int64_t row1, const leanot_wsets_t* w,
                            const double* r, double* out, double* ws, void* stream);
/* row log-normalizers L[k*nr + i] = LSE_j(-(a_k C_ij + b_kj)) (barycenter.py:78-87, core.py:67-70) */
int leanot_row_lse(const leanot_cost_t* cost, int64_t row0, int64_t row1, const leanot_wsets_t* w,
                   double* L, double* ws, void* stream);
/* _plan_stats (dxg.py:282-310) for one weight set: out3 = {<C,D_r p> (local rows), sum_i r_i H(p_i), -}, col (n) */
int leanot_plan_stats(const leanot_cost_t* cost, int64_t row0, int64_t row1, const leanot_wsets_t* w,
                      const double* r, double* col, double* out3, double* ws, void* stream);
/* row minima min_j (C_ij + v_j) (dxg.py:344-348) */
int leanot_row_min(const leanot_cost_t* cost, int64_t row0, int64_t row1, const double* v, double* out, void* stream);
/* exact-max row LSE L_i = LSE_j((sgn*C_ij + v_j)*scale): entropic dual (dxg.py:337), potentials (dxg.py:367),
 * barycenter dual (barycenter.py:189) */
int leanot_row_lse_affine(const leanot_cost_t* cost, int64_t row0, int64_t row1, const double* v, double sgn,
                          double scale, double* L, void* stream);

/* ---- the DXG solver (dxg.py:261-279, 412-472) ------------------------- */
/* derive b_bar, sd, scalars from the state (call after writing an initial/injected state).
 * init_shift: 1 = shifts from the a=0,b=0 closed form (fresh solve); 0 = compute row maxima (injected
 * state); 2 = keep the shifts left by this plan's last sweep (state produced by this plan). */
int leanot_dxg_prepare(const leanot_dxg_plan_t* plan, double a, double s, double t, int init_shift, void* stream);
/* one sweep: both column marginals of the current state into plan->col (local rows).
 * flags: LEANOT_SWEEP_EVAL accumulates evaluation statistics (rowstat); ROWS_ONLY / COLS_ONLY
 * run only pass A (row normalizers) / only pass B (column sums) so callers can time them. */
#define LEANOT_SWEEP_EVAL 1
#define LEANOT_SWEEP_ROWS_ONLY 2
#define LEANOT_SWEEP_COLS_ONLY 4
/* stored cost, plain iteration: one persistent launch, pass B re-reads C from L2
 * (csrc/leanot_fused.cu; experimental, slower than the two-pass kernels as of r01) */
#define LEANOT_SWEEP_FUSED 8
/* stored cost, plain iteration, n <= 1408 x #SMs / 2 (column tiles of the 2-group form; other
 * plans fall back to passes A + B): SINGLE_READ runs the single-read, single-exp sweep
 * (csrc/leanot_sr.cu; one read of C, one exp per element and weight set; opt-in, not faster
 * than the two-pass sweep at n = 1e5 as of r02 -- the default when LEANOT_SR=1 and n >= 32768);
 * TWO_PASS forces passes A + B */
#define LEANOT_SWEEP_TWO_PASS 16
#define LEANOT_SWEEP_SINGLE_READ 32
int leanot_dxg_sweep(const leanot_dxg_plan_t* plan, int flags, void* stream);
/* debug: device buffer of 2 x 8 x 4096 uint64 that later single-read sweeps (<= 4096 panels)
 * fill with per-panel clock64 stamps of CTAs 0 and G-1 (csrc/leanot_sr.cu); null disables
 * (the default) */
int leanot_debug_sr_trace(void* buf);
/* O(n) updates after plan->col holds the (globally reduced) marginals: state <- next state */
int leanot_dxg_update(const leanot_dxg_plan_t* plan, void* stream);
/* evaluation scalars from the last eval sweep: evalbuf[0..] = {cost_rows, ent_rows, inner_rows (eta=0 min
 * form), infeas, c.d}; eta > 0 additionally runs the LSE dual sweep (dxg.py:335-342) into S[nr, 2nr)
 * (the sweep's row minima in rowstat stay intact: repeated calls give the same scalars). */
int leanot_dxg_eval(const leanot_dxg_plan_t* plan, void* stream);
/* iters x (sweep, update) -- capturable; single process only */
int leanot_dxg_iterate(const leanot_dxg_plan_t* plan, int iters, void* stream);
/* One logging interval of solve() in one launch (small single-process plans, n <= 1024):
 * [leanot_dxg_update from the marginals of the last sweep if start_update] + the rest of
 * `iters` updates as full iterations + the evaluation sweep of the final state, i.e. the
 * sequence update / iterate / sweep(EVAL) / eval; evalbuf[0..4] as leanot_dxg_eval and
 * evalbuf[8..11] = (a, a_bar, s, t).  Returns LEANOT_EINVAL for plans it does not cover. */
int leanot_dxg_iterate_eval(const leanot_dxg_plan_t* plan, int iters, int start_update, void* stream);
/* CUDA graph of `iters` plain iterations (captured once, replayed) */
int leanot_graph_create(const leanot_dxg_plan_t* plan, int iters, void** graph_exec, void* stream);
int leanot_graph_launch(void* graph_exec, void* stream);
int leanot_graph_destroy(void* graph_exec);

/* ---- barycenter (barycenter.py:78-151) --------------------------------- */
/* Workspace of dxgb_solve / dxgb_step (barycenter.py:108-151, 227-277).  m marginals share a, s, t.
 * Per-marginal n-vectors are stacked k-major with stride ns; per-row arrays with stride nr.
 * nr = row1-row0 (= n: single-process). */
typedef struct leanot_bary_plan {
  leanot_cost_t cost;
  leanot_params_t prm;
  int64_t n, row0, row1;
  int64_t ns;            /* stride of the per-marginal n-vectors (even, >= n: 16-byte aligned slices) */
  int32_t m, splits, nblk_upd, _pad;
  const double* w;       /* m   barycenter weights (normalized) */
  const double* c;       /* m*n marginals */
  const double* c_tilde; /* m*n c_k + alpha/n */
  double* delta;         /* m*n */
  double* b;             /* m*n */
  double* b_bar;         /* m*n */
  double* bprime;        /* m*n scratch */
  double* sd;            /* m*n 2 sup tanh(delta/2) */
  double* scal;          /* 8: a, a_bar, s, t */
  int64_t* shift;        /* m*nr */
  int64_t* mu;           /* m*2*nr shifts used */
  double* S;             /* m*2*nr row sums */
  double* L;             /* 2*m*nr row log-normalizers */
  double* r;             /* 2*n  r_now | r_bar (implicit barycenters) */
  double* coef;          /* m*2*nr*4 */
  double* rowstat;       /* m*3*nr */
  double* slab;          /* splits*2*n */
  double* col;           /* m*2*n */
  double* partial;       /* >= 2*max(nblk_upd, ceil(n/256)) */
  double* scratch;       /* n */
  double* evalbuf;       /* 128 */
  int32_t* flags;        /* 2 + 4*nr */
} leanot_bary_plan_t;
int leanot_bary_prepare(const leanot_bary_plan_t* plan, double a, double s, double t, int init_shift, void* stream);
int leanot_bary_sweep(const leanot_bary_plan_t* plan, int flags, void* stream);
int leanot_bary_update(const leanot_bary_plan_t* plan, void* stream);
int leanot_bary_eval(const leanot_bary_plan_t* plan, void* stream);
/* r_i proportional to exp(sum_k w_k L_ki), k-sum in sorted order (barycenter.py:90-97);
 * scratch >= n + 2048 doubles */
int leanot_bary_rmap(const double* L, int m, int64_t n, const double* w, double* r, double* scratch, void* stream);

/* Row-sharded (multi-GPU) barycenter sweep, plan rows [row0,row1): three stream-ordered
 * phases with the caller's collectives in between (the r-map normalizers and
 * the 2 m n column partials are the only exchanges; barycenter.py:90-97, 108-151).
 *   rows:  pass A of every marginal over the plan's rows (both weight sets), the sorted k-sum
 *          g_w,i into r[w*n + i], gmax[w] = max of g_w over the plan's rows   (w = 0 now, 1 bar)
 *          -> caller: gmax = max over ranks
 *   rnorm: r_w,i = exp(g_w,i - gmax[w]), esum[w] = their sum over the plan's rows (fixed order)
 *          -> caller: esum = rank-order sum over ranks
 *   cols:  r_w,i /= esum[w], row coefficients, pass B of every marginal -> col (this rank's
 *          2 m n partials) -> caller: rank-order sum (leanot_sum_partials), then leanot_bary_update
 * gmax / esum: 2 device doubles each.  leanot_bary_eval on a sharded plan reports row sums and
 * evalbuf[127] (LSE of the dual's g) over the plan's rows; the caller combines them. */
int leanot_bary_rows(const leanot_bary_plan_t* plan, int flags, double* gmax, void* stream);
int leanot_bary_rnorm(const leanot_bary_plan_t* plan, const double* gmax, double* esum, void* stream);
int leanot_bary_cols(const leanot_bary_plan_t* plan, const double* esum, void* stream);

/* Multi-GPU combine of row-shard partials (column marginals, evaluation scalars): out[j] =
 * sum over ranks q = 0..world-1 of gathered[q*count + j], added in rank order, so every rank
 * holds bitwise-identical sums whatever the collective's internal order (the all-gather
 * replaces the reference's in-process block sum, dxg.py:205-207).  out may alias gathered. */
int leanot_sum_partials(const double* gathered, int world, int64_t count, double* out, void* stream);

/* ---- Sinkhorn / IBP baselines (sinkhorn.py:47-228) -- */
int64_t leanot_col_lse_ws_doubles(int64_t n, int64_t rows);
/* L_j = LSE_i((phi_i - C_ij)/eta) over rows [row0,row1) (sinkhorn.py:47-62); row LSEs: leanot_row_lse_affine */
int leanot_col_lse(const leanot_cost_t* cost, int64_t row0, int64_t row1, const double* phi, double eta, double* L,
                   double* ws, void* stream);
/* out = eta*log(w) - eta*L (potential update, sinkhorn.py:98) */
int leanot_eta_log_minus(const double* w, const double* L, double eta, int64_t n, double* out, void* stream);
/* psi_new = eta*log c - eta*L and gap = sum |c*expm1((psi - psi_new)/eta)| (sinkhorn.py:99-102) */
int leanot_sinkhorn_psi(const double* c, const double* L, const double* psi, double eta, int64_t n, double* psi_new,
                        double* gap, void* stream);
/* <phi,r> + <psi,c> - eta*LSE_i(phi_i/eta + L_i), L = row LSE of (psi - C)/eta (sinkhorn.py:120-136) */
int leanot_eot_dual(const double* phi, const double* psi, const double* r, const double* c, const double* L,
                    double eta, int64_t n, double* out, void* stream);
/* normalized column marginal of the plan, L = col LSE of (phi - C)/eta (sinkhorn.py:139-150) */
int leanot_sinkhorn_colmarg(const double* psi, const double* L, double eta, int64_t n, double* col, void* stream);
/* IBP shared-row step: log_r = sum_k w_k (phi_k/eta + RL_k); phi_k = eta*log_r - eta*RL_k (sinkhorn.py:222-224) */
int leanot_ibp_rows(const double* w, int m, int64_t n, double eta, const double* RL, double* phis, double* log_r,
                    void* stream);

/* ---- dense post-processing, n <= dense cap ---------- */
/* P_ij = r_i exp(-(a C_ij + b_j) - L_i), L from leanot_row_lse (materialize_plan, dxg.py:211-220) */
int leanot_materialize_plan(const leanot_cost_t* cost, double a, const double* b, const double* r, const double* L,
                            double* P, int64_t ld, void* stream);
/* Alg. 1 Round onto Pi(r, c) in place (round_to_polytope, rounding.py:63-87); scratch >= 2n+2 doubles */
int leanot_round_polytope(double* m, int64_t n, int64_t ld, const double* r, const double* c, double* scratch,
                          void* stream);
/* out[0] = <C, P> (rounded_cost, dxg.py:471); scratch >= 1024 doubles */
int leanot_plan_cost(const leanot_cost_t* cost, const double* P, int64_t ld, double* out, double* scratch,
                     void* stream);
/* pdxg_reference_step (dxg.py:494-521, the dense equivalence oracle of the reference), n <= dense cap:
 * out = z - lse_rows(z) with z = decay lp - tau (C + two_sup d[None, :]) (dxg.py:508-509, :514-515;
 * out must not alias lp), and col = r @ exp(M) (dxg.py:505-506, :511-512) */
int leanot_pdxg_rows(const leanot_cost_t* cost, const double* lp, int64_t ld, double decay, double tau, double two_sup,
                     const double* d, double* out, void* stream);
int leanot_pdxg_colsum(const double* M, int64_t n, int64_t ld, const double* r, double* col, void* stream);

/* ---- separable GridKernel path, O(n^1.5) ---------------
 * C_ij = (f(|dr|) + f(|dc|))/scale factorizes, so each n^2 LSE is two 1-D LSE convolutions.
 * The DXG sweep/eval entry points use it automatically for single-process grid plans
 * (LEANOT_GRID_SEPARABLE=0 forces the dense sweeps); the slab of such plans must hold
 * leanot_grid_sep_ws_doubles() doubles.  Each LSE convolution runs as an FP64 tensor-core
 * (DMMA) GEMM in the linear domain when its kernel table stays within e^+-600, else as an
 * exact log-domain reduction; the choice is made on device (LEANOT_SEP_GEMM=0 forces the
 * log domain). */
int64_t leanot_grid_sep_ws_doubles(const leanot_cost_t* cost);
/* L_i = LSE_j(-(a C_ij + b_j)), a in device memory; ws >= leanot_grid_sep_ws_doubles(cost) doubles */
int leanot_grid_sep_lse(const leanot_cost_t* cost, const double* a_dev, const double* b, double* L, double* ws,
                        void* stream);
/* out_z,i = LSE_j((v_z,j - C_ij)/eta) for nz potentials (rows z*vstride / z*ostride) -- the
 * Sinkhorn/IBP row (and, C being symmetric, column) LSE (sinkhorn.py:47-71);
 * ws >= leanot_grid_sep_lse_eta_ws_doubles(cost, nz) doubles */
int64_t leanot_grid_sep_lse_eta_ws_doubles(const leanot_cost_t* cost, int nz);
int leanot_grid_sep_lse_eta(const leanot_cost_t* cost, const double* v, int nz, int64_t vstride, double eta,
                            double* out, int64_t ostride, double* ws, void* stream);
/* col_j = exp(-b_j) sum_i exp(logw_i - a C_ij); ws >= leanot_grid_sep_ws_doubles(cost) doubles */
int leanot_grid_sep_colsum(const leanot_cost_t* cost, const double* a_dev, const double* b, const double* logw,
                           double* col, double* ws, void* stream);

/* stream synchronize with error capture */
int leanot_sync(void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LEANOT_B200_H */
