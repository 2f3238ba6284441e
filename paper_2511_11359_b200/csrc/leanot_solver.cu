// O(n) DXG updates, evaluation reductions, barycenter r-map, cost utilities and
// the extern "C" boundary (include/leanot_b200.h).
//
// The O(n) updates restate dxg.py:223-258 with the reference's exact operation
// order and no FMA contraction (__dmul_rn/__dadd_rn), so given identical column
// marginals the state matches NumPy to the ulp (tanh aside).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "leanot_cost.cuh"
#include "leanot_internal.h"

namespace leanot {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return LEANOT_ECUDA;
  }
  return LEANOT_OK;
}

static std::mutex g_init_mu;
static bool g_init_dev[256];

static int ensure_init() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    set_error("cudaGetDevice failed (no CUDA device?)");
    return LEANOT_ECUDA;
  }
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (dev >= 0 && dev < 256 && g_init_dev[dev]) return LEANOT_OK;
  double tab[NTAB];
  for (int j = 0; j < NTAB; ++j) {
    double v = (double)exp2l((long double)j / (long double)NTAB);
    uint64_t bits;
    memcpy(&bits, &v, 8);
    bits -= (uint64_t)j << 43;  // bias the high word by j << 11 (see leanot_common.cuh)
    memcpy(&tab[j], &bits, 8);
  }
  cudaError_t e = cudaMemcpyToSymbol(g_exp2_table, tab, sizeof(tab));
  if (e != cudaSuccess) {
    set_error("exp table upload: %s", cudaGetErrorString(e));
    return LEANOT_ECUDA;
  }
  if (dev >= 0 && dev < 256) g_init_dev[dev] = true;
  return LEANOT_OK;
}

// ---------------------------------------------------------------------------
// O(n) update kernels (dxg.py:223-258)
// ---------------------------------------------------------------------------

struct UpdArgs {
  int64_t n;
  const double* col;  // [col_now | col_bar]
  const double* c;
  const double* ct;
  double* delta;
  double* b;
  double* bprime;
  double* b_bar;
  double* sd;
  double* partial;  // 2*nblk
  double* scal;     // a, a_bar, s, t
  double A, B, beta, decay, G, twosup, tau_p, tau_p_eta;
  // batch of independent updates over blockIdx.y (barycenter marginals): element strides
  int64_t zs_col, zs_vec;  // col / (c, ct, delta, b, bprime, b_bar, sd); partial: 2 * nblk
  int nblk;
};

__device__ __forceinline__ double block_max_store(double v, double* out) {
  __shared__ double red[32];
  v = warp_max(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
    *out = t;
  }
  return v;
}

__device__ __forceinline__ double max_of(const double* p, int cnt) {
  __shared__ double red[32];
  __shared__ double res;
  double v = -INFINITY;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) v = fmax(v, p[i]);
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
    res = t;
  }
  __syncthreads();
  return res;
}

// dual_md_step(mu, col) = A*delta + (B*(col - c))/c_tilde   (dxg.py:230-232)
__device__ __forceinline__ double md_step(double A, double B, double delta, double col, double c, double ct) {
  return __dadd_rn(__dmul_rn(A, delta), __ddiv_rn(__dmul_rn(B, __dsub_rn(col, c)), ct));
}

// the update of batch member blockIdx.y
__device__ __forceinline__ UpdArgs upd_at(const UpdArgs& U0) {
  UpdArgs U = U0;
  const int64_t z = blockIdx.y;
  if (z) {
    U.col += z * U.zs_col;
    U.c += z * U.zs_vec; U.ct += z * U.zs_vec; U.delta += z * U.zs_vec; U.b += z * U.zs_vec;
    U.bprime += z * U.zs_vec; U.b_bar += z * U.zs_vec; U.sd += z * U.zs_vec;
    U.partial += z * 2 * U.nblk;
  }
  return U;
}

// K3: mu_bar, mu_next (balanced), b' = decay*b + G*tanh(mu_bar/2)  (dxg.py:273, 277-278)
__global__ void dxg_update1(const UpdArgs U0) {
  const UpdArgs U = upd_at(U0);
  double mx = -INFINITY;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < U.n; j += (int64_t)gridDim.x * blockDim.x) {
    const double cj = U.c[j], ctj = U.ct[j], dj = U.delta[j];
    const double dbar = md_step(U.A, U.B, dj, U.col[j], cj, ctj);
    double dn = md_step(U.A, U.B, dj, U.col[U.n + j], cj, ctj);
    dn = fmin(fmax(dn, -U.beta), U.beta);
    const double bp = __dadd_rn(__dmul_rn(U.decay, U.b[j]), __dmul_rn(U.G, tanh(__dmul_rn(0.5, dbar))));
    U.delta[j] = dn;
    U.bprime[j] = bp;
    mx = fmax(mx, bp);
  }
  block_max_store(mx, U.partial + blockIdx.x);
}

// K4: b = b' - max b'; then the next midpoint weights b_bar' = decay*b + G*tanh(delta/2)
//     and the dual shift sd = 2 sup tanh(delta/2)  (dxg.py:252, 274, 331-332)
__global__ void dxg_update2(const UpdArgs U0, int advance_scalars) {
  const UpdArgs U = upd_at(U0);
  const double M = max_of(U.partial, U.nblk);
  double mx = -INFINITY;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < U.n; j += (int64_t)gridDim.x * blockDim.x) {
    const double bn = __dsub_rn(U.bprime[j], M);
    const double d = tanh(__dmul_rn(0.5, U.delta[j]));
    const double bb = __dadd_rn(__dmul_rn(U.decay, bn), __dmul_rn(U.G, d));
    U.b[j] = bn;
    U.sd[j] = __dmul_rn(U.twosup, d);
    U.bprime[j] = bb;
    mx = fmax(mx, bb);
  }
  block_max_store(mx, U.partial + U.nblk + blockIdx.x);
  if (advance_scalars && blockIdx.x == 0 && blockIdx.y == gridDim.y - 1 && threadIdx.x == 0) {
    // TransportLogWeights(a, s, t) advance (dxg.py:253-257) and the next midpoint a
    const double a = __dadd_rn(__dmul_rn(U.decay, U.scal[0]), U.tau_p);
    U.scal[0] = a;
    U.scal[1] = __dadd_rn(__dmul_rn(U.decay, a), U.tau_p);
    U.scal[2] = __dadd_rn(__dmul_rn(U.decay, U.scal[2]), U.tau_p_eta);
    U.scal[3] = U.scal[3] + 1.0;
  }
}

// Small n (launch-bound): K3 + K4 + K5 in one CTA on the reduced columns (same arithmetic,
// same order of operations per element; maxima are order-independent).
__global__ void __launch_bounds__(1024) dxg_update_small(const UpdArgs U) {
  __shared__ double red[32];
  __shared__ double bc;
  const int64_t n = U.n;
  auto bmax = [&](double v) -> double {
    v = warp_max(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
      bc = t;
    }
    __syncthreads();
    const double r = bc;
    __syncthreads();
    return r;
  };
  double mx = -INFINITY;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const double cn = U.col[j], cb = U.col[n + j];
    const double cj = U.c[j], ctj = U.ct[j], dj = U.delta[j];
    const double dbar = md_step(U.A, U.B, dj, cn, cj, ctj);
    double dn = md_step(U.A, U.B, dj, cb, cj, ctj);
    dn = fmin(fmax(dn, -U.beta), U.beta);
    const double bp = __dadd_rn(__dmul_rn(U.decay, U.b[j]), __dmul_rn(U.G, tanh(__dmul_rn(0.5, dbar))));
    U.delta[j] = dn;
    U.bprime[j] = bp;
    mx = fmax(mx, bp);
  }
  const double M = bmax(mx);
  mx = -INFINITY;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const double bn = __dsub_rn(U.bprime[j], M);
    const double d = tanh(__dmul_rn(0.5, U.delta[j]));
    const double bb = __dadd_rn(__dmul_rn(U.decay, bn), __dmul_rn(U.G, d));
    U.b[j] = bn;
    U.sd[j] = __dmul_rn(U.twosup, d);
    U.bprime[j] = bb;
    mx = fmax(mx, bb);
  }
  const double Mb = bmax(mx);
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) U.b_bar[j] = __dsub_rn(U.bprime[j], Mb);
  if (threadIdx.x == 0) {
    const double a = __dadd_rn(__dmul_rn(U.decay, U.scal[0]), U.tau_p);
    U.scal[0] = a;
    U.scal[1] = __dadd_rn(__dmul_rn(U.decay, a), U.tau_p);
    U.scal[2] = __dadd_rn(__dmul_rn(U.decay, U.scal[2]), U.tau_p_eta);
    U.scal[3] = U.scal[3] + 1.0;
  }
}

// K5: b_bar = b_bar' - max b_bar'
__global__ void dxg_update3(const UpdArgs U0) {
  const UpdArgs U = upd_at(U0);
  const double M = max_of(U.partial + U.nblk, U.nblk);
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < U.n; j += (int64_t)gridDim.x * blockDim.x)
    U.b_bar[j] = __dsub_rn(U.bprime[j], M);
}

// prepare from a state: sd, b_bar' and scalars (a, s, t given by the host)
__global__ void dxg_prepare_kernel(const UpdArgs U, double a, double s, double t) {
  double mx = -INFINITY;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < U.n; j += (int64_t)gridDim.x * blockDim.x) {
    const double d = tanh(__dmul_rn(0.5, U.delta[j]));
    const double bb = __dadd_rn(__dmul_rn(U.decay, U.b[j]), __dmul_rn(U.G, d));
    U.sd[j] = __dmul_rn(U.twosup, d);
    U.bprime[j] = bb;
    mx = fmax(mx, bb);
  }
  block_max_store(mx, U.partial + U.nblk + blockIdx.x);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    U.scal[0] = a;
    U.scal[1] = __dadd_rn(__dmul_rn(U.decay, a), U.tau_p);
    U.scal[2] = s;
    U.scal[3] = t;
  }
}

__global__ void fill_i64_kernel(int64_t* p, int64_t cnt, int64_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void max_i64_pair_kernel(const int64_t* a, const int64_t* b, int64_t* out, int64_t cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] > b[i] ? a[i] : b[i];
}

// ---------------------------------------------------------------------------
// evaluation reductions (single CTA, fixed order -> deterministic)
// ---------------------------------------------------------------------------

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double red[32];
  __shared__ double res;
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    res = t;
  }
  __syncthreads();
  double out = res;
  __syncthreads();
  return out;
}

// Row part of _evaluate for weight set 0 of the last evaluation sweep:
//   out[0] = sum_i (r_i/S_i) sum_j e_ij C_ij          = <C, D_r p>     (dxg.py:295)
//   out[1] = sum_i r_i (L_i - sum_j p_ij x_ij)       = sum r_i H(p_i) (dxg.py:298-299)
//   out[2] = sum_i r_i v_i  (v = row min, or the dual row LSE)        (dxg.py:342/348)
__global__ void rowstats_reduce_kernel(int64_t nr, int64_t row0, const double* r, const double* S, const int64_t* m,
                                       const double* rowstat, const double* v, double* out) {
  double cst = 0.0, ent = 0.0, inner = 0.0;
  for (int64_t li = threadIdx.x; li < nr; li += blockDim.x) {
    const double ri = r[row0 + li];
    const double Si = S[li];
    cst += (ri / Si) * rowstat[li];
    if (ri > 0.0) {
      const double L = (double)m[li] * LSTEP + log(Si);
      ent += ri * (L - rowstat[nr + li] / Si);
    }
    if (v) inner += ri * v[li];
  }
  cst = block_sum(cst);
  ent = block_sum(ent);
  inner = block_sum(inner);
  if (threadIdx.x == 0) { out[0] = cst; out[1] = ent; out[2] = inner; }
}

// Column part: out[0] = ||col - c||_1 (dxg.py:414), out[1] = <c, tanh(delta/2)> (dxg.py:349)
__global__ void colstats_reduce_kernel(int64_t n, const double* col, const double* c, const double* delta, double* out) {
  double inf = 0.0, cd = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    inf += fabs(col[j] - c[j]);
    if (delta) cd += c[j] * tanh(0.5 * delta[j]);
  }
  inf = block_sum(inf);
  cd = block_sum(cd);
  if (threadIdx.x == 0) { out[0] = inf; out[1] = cd; }
}

// ---------------------------------------------------------------------------
// barycenter r-map (barycenter.py:90-97): g_i = sorted_k(w_k L_ki) summed in
// ascending order, r = exp(g - max g) / sum
// ---------------------------------------------------------------------------

__global__ void bary_g_kernel(const double* L, int m, int64_t n, const double* w, double* g, double* partial) {
  double mx = -INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v[LEANOT_MAX_K];
    for (int k = 0; k < m; ++k) v[k] = w[k] * L[k * n + i];
    for (int a = 1; a < m; ++a) {  // insertion sort (m <= 16), NaN-free inputs
      double x = v[a];
      int b = a - 1;
      while (b >= 0 && v[b] > x) { v[b + 1] = v[b]; --b; }
      v[b + 1] = x;
    }
    double s = v[0];
    for (int k = 1; k < m; ++k) s += v[k];
    g[i] = s;
    mx = fmax(mx, s);
  }
  block_max_store(mx, partial + blockIdx.x);
}

// e_i = exp(g_i - max g) and per-block partial sums (partial[0..nblk) holds the block maxima)
__global__ void bary_e_kernel(const double* g, int64_t n, const double* partial, int nblk, double* r, double* psum) {
  const double M = max_of(partial, nblk);
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double e = exp(g[i] - M);
    r[i] = e;
    s += e;
  }
  s = block_sum(s);
  if (threadIdx.x == 0) psum[blockIdx.x] = s;
}

// r_i /= sum of the block partial sums; every block adds them with the same fixed tree
// (strided per-thread sums, then block_sum), so all blocks divide by the identical total
__global__ void bary_norm_kernel(double* r, int64_t n, const double* psum, int nblk) {
  __shared__ double tot;
  double t = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) t += psum[b];
  t = block_sum(t);
  if (threadIdx.x == 0) tot = t;
  __syncthreads();
  const double s = tot;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = r[i] / s;
}

// out = sum of p[0..cnt) in a fixed order (strided per-thread sums, then block_sum)
__global__ void sum_fixed_kernel(const double* p, int cnt, double* out) {
  double t = 0.0;
  for (int q = threadIdx.x; q < cnt; q += blockDim.x) t += p[q];
  t = block_sum(t);
  if (threadIdx.x == 0) out[0] = t;
}

// full r-map over all SMs; partial needs 2 * nblk doubles (nblk <= 1024)
static void launch_rmap(const double* L, int m, int64_t n, const double* w, double* g, double* partial, double* r,
                        cudaStream_t st) {
  const int nblk = (int)std::min<int64_t>((n + 255) / 256, 1024);
  bary_g_kernel<<<nblk, 256, 0, st>>>(L, m, n, w, g, partial);
  bary_e_kernel<<<nblk, 256, 0, st>>>(g, n, partial, nblk, r, partial + nblk);
  bary_norm_kernel<<<nblk, 256, 0, st>>>(r, n, partial + nblk, nblk);
}

// ---------------------------------------------------------------------------
// cost utilities
// ---------------------------------------------------------------------------

__global__ void stored_max_kernel(const double* mat, int64_t rows, int64_t cols, int64_t ld, double* partial) {
  double mx = -INFINITY;
  for (int64_t i = blockIdx.x; i < rows; i += gridDim.x)
    for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) mx = fmax(mx, mat[i * ld + j]);
  block_max_store(mx, partial + blockIdx.x);
}

__global__ void stored_min_kernel(const double* mat, int64_t rows, int64_t cols, int64_t ld, double* partial) {
  double mn = INFINITY;
  for (int64_t i = blockIdx.x; i < rows; i += gridDim.x)
    for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) mn = fmin(mn, mat[i * ld + j]);
  block_max_store(-mn, partial + blockIdx.x);
}

__global__ void reduce_max_kernel(const double* partial, int cnt, double* out) {
  const double M = max_of(partial, cnt);
  if (threadIdx.x == 0) *out = M;
}

__global__ void stored_normalize_kernel(double* mat, int64_t rows, int64_t cols, int64_t ld, double scale) {
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y)
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cols; j += (int64_t)gridDim.x * blockDim.x)
      mat[i * ld + j] = mat[i * ld + j] / scale;
}

__device__ __forceinline__ uint64_t splitmix(uint64_t key, uint64_t seed) {
  uint64_t z = key ^ (seed * 0x9E3779B97F4A7C15ull);
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// C_ij = U[0,1) (splitmix64 of (i<<32|j) ^ seed*golden), C[0][n-1] = 1 (oracle/leanot_oracle.py:hash_u01)
__global__ void hash_fill_kernel(double* mat, int64_t row0, int64_t rows, int64_t n, int64_t ld, uint64_t seed) {
  for (int64_t li = blockIdx.y; li < rows; li += gridDim.y) {
    const uint64_t i = (uint64_t)(row0 + li);
    for (int64_t j = 2 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); j < n; j += 2 * (int64_t)gridDim.x * blockDim.x) {
      double v0 = (double)(splitmix((i << 32) | (uint64_t)j, seed) >> 11) * 0x1p-53;
      double v1 = 0.0;
      if (j + 1 < n) v1 = (double)(splitmix((i << 32) | (uint64_t)(j + 1), seed) >> 11) * 0x1p-53;
      if (i == 0 && j + 1 == n - 1) v1 = 1.0;
      if (i == 0 && j == n - 1) v0 = 1.0;
      if (j + 1 < ld) {
        *reinterpret_cast<double2*>(mat + li * ld + j) = make_double2(v0, v1);
      } else {
        mat[li * ld + j] = v0;
      }
    }
  }
}

// out[j] = sum of the world ranks' partials in rank order (engine.combine_partials)
__global__ void sum_partials_kernel(const double* g, int world, int64_t count, double* out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < count; j += (int64_t)gridDim.x * blockDim.x) {
    double s = g[j];
    for (int q = 1; q < world; ++q) s += g[(int64_t)q * count + j];
    out[j] = s;
  }
}

// beta_kj = -a_k inv N_j - b_kj for the expanded-form sweeps (CostGram), k = 0 (b), 1 (b_bar)
__global__ void gram_beta_kernel(int64_t n, int64_t ld, const double* scal, double inv, const double* N,
                                 const double* b, const double* bb, double* beta) {
  const double na0 = (-scal[0]) * inv, na1 = (-scal[1]) * inv;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double Nj = N[j];
    beta[j] = fma(na0, Nj, -b[j]);
    beta[ld + j] = fma(na1, Nj, -bb[j]);
  }
}

// Expanded (Gram) form of squared-Euclidean costs.  |f_i - f_j|^2 does not change under a
// translation, so the form runs on features centered at their mean mu: the cancellation in
// N_i + N_j - 2 f_i.f_j then costs ~ulp(|f - mu|^2) instead of ulp(|f|^2) (point clouds far
// from the origin).  One CTA computes mu per dimension in a fixed order (deterministic).
__global__ void __launch_bounds__(1024) points_mean_kernel(const double* f, int64_t n, int dim, double* mu) {
  __shared__ double red[32][4];
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x)
    for (int d = 0; d < dim; ++d) s[d] += f[j * dim + d];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = 0; d < dim; ++d) {
    const double v = warp_sum(s[d]);
    if (lane == 0) red[warp][d] = v;
  }
  __syncthreads();
  if (threadIdx.x < dim) {
    double t = red[0][threadIdx.x];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t += red[w][threadIdx.x];
    mu[threadIdx.x] = t / (double)n;
  }
}

// out[j] = |f_j - mu|^2 (j < n), out[np + j*dim + d] = f_jd - mu_d (np = n rounded up to even)
__global__ void points_norms_kernel(const double* f, int64_t n, int dim, const double* mu, double* out) {
  const int64_t np = (n + 1) & ~int64_t(1);
  double m[4];
  for (int d = 0; d < dim; ++d) m[d] = mu[d];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double g0 = f[j * dim] - m[0];
    out[np + j * dim] = g0;
    double s = g0 * g0;
    for (int d = 1; d < dim; ++d) {
      const double g = f[j * dim + d] - m[d];
      out[np + j * dim + d] = g;
      s = fma(g, g, s);
    }
    out[j] = s;
  }
}

__global__ void points_sup_kernel(const double* f, int64_t n, int dim, int p, double* partial) {
  double mx = 0.0;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      double s = 0.0;
      for (int d = 0; d < dim; ++d) {
        double dd = fabs(f[i * dim + d] - f[j * dim + d]);
        s += p == 1 ? dd : (p == 2 ? dd * dd : dd * dd * dd);
      }
      mx = fmax(mx, s);
    }
  }
  block_max_store(mx, partial + blockIdx.x);
}

static cudaStream_t S_(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static UpdArgs make_upd(const leanot_dxg_plan_t& P) {
  UpdArgs U;
  U.n = P.n; U.col = P.col; U.c = P.c; U.ct = P.c_tilde; U.delta = P.delta; U.b = P.b; U.bprime = P.bprime;
  U.b_bar = P.b_bar; U.sd = P.sd; U.partial = P.partial; U.scal = P.scal;
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
  U.zs_col = 0;
  U.zs_vec = 0;
  return U;
}

// separable grid path (leanot_sep.cu)
static bool use_sep(const leanot_dxg_plan_t& P);
static int sep_dxg_sweep(const leanot_dxg_plan_t& P, bool eval, cudaStream_t st);
static int sep_dxg_eval(const leanot_dxg_plan_t& P, cudaStream_t st);
// persistent small-n iterations (leanot_persist.cu)
static int try_persist_iterate(const leanot_dxg_plan_t& P, int iters, cudaStream_t st);
static int try_rowowner_iterate_eval(const leanot_dxg_plan_t& P, int iters, int start_update, cudaStream_t st);
// single-launch L2-reuse sweep for stored costs (leanot_fused.cu)
static int try_fused_sweep(const leanot_dxg_plan_t& P, cudaStream_t st);
static bool fused_default();
// single-read, single-exp sweep for stored costs (leanot_sr.cu)
static int try_sr_sweep(const leanot_dxg_plan_t& P, cudaStream_t st, bool force);

// plans whose O(n) work fits one CTA and whose sweep covers all rows (single process):
// launch-bound regime, fused update path (reduces the column slabs itself)
// One-CTA update (dxg_update_small) up to this n; above it the three grid-wide kernels.
// The single CTA is FP64-bound on its two divisions and two tanh per element: measured in
// CUDA-graph replays (tools/upd_ab.py), the grid-wide kernels win from n ~ 5000 on
// (n = 1e4: 370 -> 360 us per iteration; n = 3000: the single CTA is 2 us faster).
// LEANOT_SMALL_UPD_N overrides (A/B measurements).
static int64_t small_upd_max_n() {
  static int64_t v = -1;
  if (v < 0) {
    const char* e = getenv("LEANOT_SMALL_UPD_N");
    v = e ? atoll(e) : 4096;
  }
  return v;
}

static bool small_plan(const leanot_dxg_plan_t& P) {
  return P.n <= small_upd_max_n() && P.row0 == 0 && P.row1 == P.n && !use_sep(P);
}

static RowPassArgs make_rowpass(const leanot_dxg_plan_t& P) {
  RowPassArgs A;
  memset(&A, 0, sizeof(A));
  A.cost = make_view(P.cost);
  A.i0 = P.row0; A.i1 = P.row1;
  A.a = P.scal;
  A.b[0] = P.b; A.b[1] = P.b_bar;
  A.shift = P.shift; A.shift_kstride = 0;
  A.S = P.S; A.m_used = P.m;
  A.rowstat = P.rowstat; A.sd = P.sd;
  A.rw = P.r; A.coef = P.coef;
  A.shift_next = P.shift; A.next_from_k = 1;
  A.flags = P.flags;
  return A;
}

static int validate_cost(const leanot_cost_t* c) {
  if (!c) { set_error("null cost"); return LEANOT_EINVAL; }
  if (c->n < 1) { set_error("cost n must be positive"); return LEANOT_EINVAL; }
  if (c->kind == LEANOT_COST_STORED) {
    if (!c->mat || c->ld < c->n || (c->ld & 1) || (reinterpret_cast<uintptr_t>(c->mat) & 15)) {
      set_error("stored cost needs a 16-byte aligned matrix with even ld >= n");
      return LEANOT_EINVAL;
    }
  } else if (c->kind == LEANOT_COST_POINTS) {
    if (!c->feat || c->dim < 1 || c->dim > 4 || c->p < 1 || c->p > 3 || (reinterpret_cast<uintptr_t>(c->feat) & 15)) {
      set_error("points cost needs 16-byte aligned features with 1 <= dim <= 4 and p in {1,2,3}");
      return LEANOT_EINVAL;
    }
  } else if (c->kind == LEANOT_COST_GRID) {
    if (!c->grid_coords || c->p < 1 || c->p > 3 || (int64_t)c->height * c->width != c->n) {
      set_error("grid cost needs coordinates, p in {1,2,3} and height*width == n");
      return LEANOT_EINVAL;
    }
  } else {
    set_error("unknown cost kind %d", c->kind);
    return LEANOT_EINVAL;
  }
  return LEANOT_OK;
}

#define LEANOT_TRY(x)              \
  do {                             \
    int _rc = (x);                 \
    if (_rc != LEANOT_OK) return _rc; \
  } while (0)

}  // namespace leanot

using namespace leanot;

extern "C" {

int leanot_version(void) { return LEANOT_ABI_VERSION; }

const char* leanot_last_error(void) { return g_err; }

int leanot_device_sm_count(int device, int* out) {
  int v = 0;
  cudaError_t e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); return LEANOT_ECUDA; }
  *out = v;
  return LEANOT_OK;
}

int leanot_dxg_default_splits(int64_t n, int64_t rows, int* out) {
  // column pass work items = ceil(n/512) tiles x splits; aim for >= 2 waves of 3 CTAs/SM
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (n + 1023) / 1024;   // column-pass tile = 1024 columns
  const int64_t smax = std::min<int64_t>(64, std::max<int64_t>(1, rows / 8));
  if (n <= 16384 || n >= 262144) {
    // small plans and very large ones: the column pass is a few waves of (tile, split) items over the 2 x SMs
    // resident CTAs, so pick the split count whose items fill the last wave best (fewest
    // items among the best); at n = 1e4 this is 29 splits = 290 items in one wave, 11 %
    // faster than 64 splits = 2.16 waves (tools/splits_sweep.py)
    const int64_t G = (int64_t)sms * 2;
    auto eff_of = [&](int64_t s) {
      const int64_t items = tiles * s;
      return (double)items / (double)(((items + G - 1) / G) * G);
    };
    // >= ~one wave for small n; >= 3 waves for the large on-the-fly shards (BASELINE config 4:
    // 3 splits = 9.9 waves, pass B 5 % faster than 2 splits = 6.6 waves)
    const int64_t min_items = n <= 16384 ? (G * 9) / 10 : 3 * G;
    auto eligible = [&](int64_t s) { return tiles * s >= min_items || s == smax; };
    double best_eff = 0.0;
    for (int64_t s = 1; s <= smax; ++s)
      if (eligible(s)) best_eff = std::max(best_eff, eff_of(s));
    int64_t best = smax;
    for (int64_t s = 1; s <= smax; ++s)
      if (eligible(s) && eff_of(s) >= best_eff - 0.02) { best = s; break; }
    *out = (int)best;
    return LEANOT_OK;
  }
  const int64_t target = (int64_t)sms * 3 * 4;  // >= 4 work items per resident CTA
  int64_t s = (target + tiles - 1) / tiles;
  s = std::max<int64_t>(1, std::min<int64_t>(s, smax));
  *out = (int)s;
  return LEANOT_OK;
}

int leanot_cost_block(const leanot_cost_t* cost, int64_t i0, int64_t i1, double* out, int64_t ldo, void* stream) {
  LEANOT_TRY(validate_cost(cost));
  LEANOT_TRY(ensure_init());
  if (i0 < 0 || i1 > cost->n || i0 > i1 || ldo < cost->n) { set_error("bad block range"); return LEANOT_EINVAL; }
  LEANOT_TRY(launch_cost_block(make_view(*cost), i0, i1, out, ldo, S_(stream)));
  return check_launch("cost_block");
}

int leanot_stored_max(const double* mat, int64_t rows, int64_t cols, int64_t ld, double* out, double* scratch, void* stream) {
  LEANOT_TRY(ensure_init());
  int grid = (int)std::min<int64_t>(std::max<int64_t>(rows, 1), 1024);
  stored_max_kernel<<<grid, 256, 0, S_(stream)>>>(mat, rows, cols, ld, scratch);
  reduce_max_kernel<<<1, 1024, 0, S_(stream)>>>(scratch, grid, out);
  stored_min_kernel<<<grid, 256, 0, S_(stream)>>>(mat, rows, cols, ld, scratch + 1024);
  reduce_max_kernel<<<1, 1024, 0, S_(stream)>>>(scratch + 1024, grid, out + 1);  // out[1] = -min
  return check_launch("stored_max");
}

int leanot_stored_normalize(double* mat, int64_t rows, int64_t cols, int64_t ld, double scale, void* stream) {
  LEANOT_TRY(ensure_init());
  if (!(scale > 0)) { set_error("scale must be positive"); return LEANOT_EINVAL; }
  dim3 grid((unsigned)std::min<int64_t>((cols + 255) / 256, 32), (unsigned)std::min<int64_t>(std::max<int64_t>(rows, 1), 8192));
  stored_normalize_kernel<<<grid, 256, 0, S_(stream)>>>(mat, rows, cols, ld, scale);
  return check_launch("stored_normalize");
}

int leanot_points_sup(const double* feat, int64_t n, int dim, int p, double* out, double* scratch, void* stream) {
  LEANOT_TRY(ensure_init());
  int grid = (int)std::min<int64_t>(std::max<int64_t>(n, 1), 1024);
  points_sup_kernel<<<grid, 256, 0, S_(stream)>>>(feat, n, dim, p, scratch);
  reduce_max_kernel<<<1, 1024, 0, S_(stream)>>>(scratch, grid, out);
  return check_launch("points_sup");
}

int leanot_points_norms(const double* feat, int64_t n, int dim, double* out, void* stream) {
  LEANOT_TRY(ensure_init());
  if (!feat || !out || n < 1 || dim < 1 || dim > 4) { set_error("points_norms: bad arguments"); return LEANOT_EINVAL; }
  // out = [|f_j - mu|^2 (n, padded to even) | f_j - mu (n x dim) | mu (dim)]
  double* mu = out + ((n + 1) & ~int64_t(1)) + n * dim;
  points_mean_kernel<<<1, 1024, 0, S_(stream)>>>(feat, n, dim, mu);
  points_norms_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, S_(stream)>>>(feat, n, dim, mu, out);
  return check_launch("points_norms");
}

int leanot_sum_partials(const double* gathered, int world, int64_t count, double* out, void* stream) {
  LEANOT_TRY(ensure_init());
  if (!gathered || !out || world < 1 || count < 0) { set_error("sum_partials: bad arguments"); return LEANOT_EINVAL; }
  if (count == 0) return LEANOT_OK;
  sum_partials_kernel<<<(int)std::min<int64_t>((count + 255) / 256, 4096), 256, 0, S_(stream)>>>(gathered, world, count,
                                                                                                 out);
  return check_launch("sum_partials");
}

int leanot_hash_fill(double* mat, int64_t row0, int64_t rows, int64_t n, int64_t ld, uint64_t seed, void* stream) {
  LEANOT_TRY(ensure_init());
  if ((ld & 1) || ld < n) { set_error("hash_fill needs even ld >= n"); return LEANOT_EINVAL; }
  dim3 grid((unsigned)std::min<int64_t>((n / 2 + 255) / 256 + 1, 64), (unsigned)std::min<int64_t>(std::max<int64_t>(rows, 1), 16384));
  hash_fill_kernel<<<grid, 256, 0, S_(stream)>>>(mat, row0, rows, n, ld, seed);
  return check_launch("hash_fill");
}

int64_t leanot_sweep_ws_doubles(int64_t n, int64_t rows, int K) {
  int splits = 1;
  leanot_dxg_default_splits(n, rows, &splits);
  // shift(rows) + m(K rows) + S(K rows) + coef(4K rows) + slab(splits K n) + flags(2+2K rows ints) + stats(3 rows) + 16
  return rows + K * rows + K * rows + 4 * K * rows + (int64_t)splits * K * n + (2 + 2 * K * rows + 1) / 2 + 1 +
         3 * rows + 16;
}

struct SweepWs {
  int64_t* shift;
  int64_t* m;
  double* S;
  double* coef;
  double* slab;
  int32_t* flags;
  double* stats;
  double* misc;
  int splits;
};

static SweepWs carve_ws(double* ws, int64_t n, int64_t rows, int K) {
  SweepWs w;
  leanot_dxg_default_splits(n, rows, &w.splits);
  double* p = ws;
  w.shift = reinterpret_cast<int64_t*>(p); p += rows;
  w.m = reinterpret_cast<int64_t*>(p); p += K * rows;
  w.S = p; p += K * rows;
  w.coef = p; p += 4 * K * rows;
  w.slab = p; p += (int64_t)w.splits * K * n;
  w.flags = reinterpret_cast<int32_t*>(p); p += (2 + 2 * K * rows + 1) / 2 + 1;
  w.stats = p; p += 3 * rows;
  w.misc = p;
  return w;
}

// shared robust start + pass A + pass B for K independent weight sets (K <= 2)
static int sweep_k(const leanot_cost_t* cost, int64_t row0, int64_t row1, const leanot_wsets_t* w, const double* r,
                   double* colout, double* ws, bool eval, const double* sd, cudaStream_t st, SweepWs* outw) {
  const int64_t n = cost->n, nr = row1 - row0;
  const int K = w->K;
  SweepWs W = carve_ws(ws, n, nr, K);
  if (outw) *outw = W;
  cudaMemsetAsync(W.flags, 0, 8, st);
  RowPassArgs A;
  memset(&A, 0, sizeof(A));
  A.cost = make_view(*cost);
  A.i0 = row0; A.i1 = row1;
  A.a = w->a;
  for (int k = 0; k < K; ++k) A.b[k] = w->b[k];
  A.shift = W.shift; A.shift_kstride = 0;
  A.S = W.S; A.m_used = W.m;
  A.rowstat = W.stats; A.sd = sd;
  A.rw = r; A.coef = W.coef;
  A.flags = W.flags;
  // robust shift: max over weight sets of the row maxima
  LEANOT_TRY(launch_rowmax(A, K, W.m, st));
  if (K == 2) {
    max_i64_pair_kernel<<<(int)std::min<int64_t>((nr + 255) / 256, 1024), 256, 0, st>>>(W.m, W.m + nr, W.shift, nr);
  } else {
    cudaMemcpyAsync(W.shift, W.m, nr * sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
  }
  LEANOT_TRY(launch_rowpass(A, K, eval, st));
  if (colout) {
    ColPassArgs B;
    memset(&B, 0, sizeof(B));
    B.cost = A.cost; B.i0 = row0; B.i1 = row1; B.a = w->a;
    for (int k = 0; k < K; ++k) B.b[k] = w->b[k];
    B.m = W.m; B.coef = W.coef; B.slab = W.slab; B.splits = W.splits;
    LEANOT_TRY(launch_colpass(B, K, st));
    LEANOT_TRY(launch_slab_reduce(W.slab, W.splits, K, n, colout, st));
  }
  return LEANOT_OK;
}

int leanot_column_marginals(const leanot_cost_t* cost, int64_t row0, int64_t row1, const leanot_wsets_t* w,
                            const double* r, double* out, double* ws, void* stream) {
  LEANOT_TRY(validate_cost(cost));
  LEANOT_TRY(ensure_init());
  if (!w || w->K < 1 || w->K > 2) { set_error("column_marginals supports K in {1,2}"); return LEANOT_EINVAL; }
  if (row0 < 0 || row1 > cost->n || row0 >= row1) { set_error("bad row range"); return LEANOT_EINVAL; }
  LEANOT_TRY(sweep_k(cost, row0, row1, w, r, out, ws, false, nullptr, S_(stream), nullptr));
  return check_launch("column_marginals");
}

__global__ void lse_from_sums_kernel(const int64_t* m, const double* S, int64_t cnt, double* L) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
    L[i] = (double)m[i] * LSTEP + log(S[i]);
}

int leanot_row_lse(const leanot_cost_t* cost, int64_t row0, int64_t row1, const leanot_wsets_t* w, double* L, double* ws,
                   void* stream) {
  LEANOT_TRY(validate_cost(cost));
  LEANOT_TRY(ensure_init());
  if (!w || w->K < 1 || w->K > LEANOT_MAX_K) { set_error("bad weight sets"); return LEANOT_EINVAL; }
  const int64_t nr = row1 - row0;
  for (int k = 0; k < w->K; ++k) {
    leanot_wsets_t one;
    memset(&one, 0, sizeof(one));
    one.K = 1; one.a = w->a + k; one.b[0] = w->b[k];
    SweepWs W;
    LEANOT_TRY(sweep_k(cost, row0, row1, &one, nullptr, nullptr, ws, false, nullptr, S_(stream), &W));
    lse_from_sums_kernel<<<(int)std::min<int64_t>((nr + 255) / 256, 1024), 256, 0, S_(stream)>>>(W.m, W.S, nr, L + k * nr);
  }
  return check_launch("row_lse");
}

int leanot_plan_stats(const leanot_cost_t* cost, int64_t row0, int64_t row1, const leanot_wsets_t* w, const double* r,
                      double* col, double* out3, double* ws, void* stream) {
  LEANOT_TRY(validate_cost(cost));
  LEANOT_TRY(ensure_init());
  if (!w || w->K != 1) { set_error("plan_stats takes one weight set"); return LEANOT_EINVAL; }
  const int64_t nr = row1 - row0;
  SweepWs W;
  // the eval sweep also tracks a row min against `sd`; reuse b as a harmless vector
  LEANOT_TRY(sweep_k(cost, row0, row1, w, r, col, ws, true, w->b[0], S_(stream), &W));
  rowstats_reduce_kernel<<<1, 1024, 0, S_(stream)>>>(nr, row0, r, W.S, W.m, W.stats, nullptr, out3);
  return check_launch("plan_stats");
}

int leanot_row_min(const leanot_cost_t* cost, int64_t row0, int64_t row1, const double* v, double* out, void* stream) {
  LEANOT_TRY(validate_cost(cost));
  LEANOT_TRY(ensure_init());
  LEANOT_TRY(launch_rowmin(make_view(*cost), row0, row1, v, out, S_(stream)));
  return check_launch("row_min");
}

int leanot_row_lse_affine(const leanot_cost_t* cost, int64_t row0, int64_t row1, const double* v, double sgn, double scale,
                          double* L, void* stream) {
  LEANOT_TRY(validate_cost(cost));
  LEANOT_TRY(ensure_init());
  LEANOT_TRY(launch_rowlse(make_view(*cost), row0, row1, v, sgn, scale, L, S_(stream)));
  return check_launch("row_lse_affine");
}

// ---- solver -----------------------------------------------------------------

static int validate_plan(const leanot_dxg_plan_t* P) {
  if (!P) { set_error("null plan"); return LEANOT_EINVAL; }
  LEANOT_TRY(validate_cost(&P->cost));
  if (P->n != P->cost.n || P->row0 < 0 || P->row1 > P->n || P->row0 >= P->row1 || P->splits < 1 || P->nblk_upd < 1 ||
      P->nblk_upd > 1024) {
    set_error("inconsistent plan sizes");
    return LEANOT_EINVAL;
  }
  return LEANOT_OK;
}

int leanot_dxg_prepare(const leanot_dxg_plan_t* P, double a, double s, double t, int init_shift, void* stream) {
  LEANOT_TRY(validate_plan(P));
  LEANOT_TRY(ensure_init());
  cudaStream_t st = S_(stream);
  UpdArgs U = make_upd(*P);
  dxg_prepare_kernel<<<P->nblk_upd, 256, 0, st>>>(U, a, s, t);
  dxg_update3<<<P->nblk_upd, 256, 0, st>>>(U);
  cudaMemsetAsync(P->flags, 0, 8, st);
  const int64_t nr = P->row1 - P->row0;
  if (init_shift == 2) {
    // keep the shifts the last sweep of this plan left behind (warm restart of the
    // state it produced; any shift is valid -- rows out of range are recomputed)
  } else if (init_shift) {
    // a = 0, b = 0: x = 0 and L = log n for every row (the midpoint set is within tau_p)
    fill_i64_kernel<<<(int)std::min<int64_t>((nr + 255) / 256, 1024), 256, 0, st>>>(
        P->shift, nr, llrint(log((double)P->n) * (1.0 / LSTEP)));
  } else {
    RowPassArgs A = make_rowpass(*P);
    LEANOT_TRY(launch_rowmax(A, 2, P->m, st));
    max_i64_pair_kernel<<<(int)std::min<int64_t>((nr + 255) / 256, 1024), 256, 0, st>>>(P->m, P->m + nr, P->shift, nr);
  }
  return check_launch("dxg_prepare");
}

int leanot_dxg_sweep(const leanot_dxg_plan_t* P, int flags, void* stream) {
  LEANOT_TRY(validate_plan(P));
  LEANOT_TRY(ensure_init());
  cudaStream_t st = S_(stream);
  if (use_sep(*P)) {
    // grid cost: O(n^1.5) separable sweep (both phases at once; phase flags ignored)
    if (flags & LEANOT_SWEEP_ROWS_ONLY) return LEANOT_OK;
    LEANOT_TRY(sep_dxg_sweep(*P, (flags & LEANOT_SWEEP_EVAL) != 0, st));
    return check_launch("dxg_sweep(separable)");
  }
  RowPassArgs A = make_rowpass(*P);
  // squared-Euclidean points: expanded form for the plain iteration sweeps (the evaluation
  // sweep needs C itself); pass A and pass B must agree (shift / coefficient convention)
  const bool eval = (flags & LEANOT_SWEEP_EVAL) != 0;
  const bool gram = !eval && P->beta && P->cost.kind == LEANOT_COST_POINTS && P->cost.p == 2 && P->cost.norms &&
                    gram_enabled();
  if (gram) {
    A.gram = 1;
    const int64_t ld = (P->n + 1) & ~int64_t(1);  // beta_1 16-byte aligned (pass A reads double2)
    A.b[0] = P->beta; A.b[1] = P->beta + ld;
    if (!(flags & LEANOT_SWEEP_COLS_ONLY))
      gram_beta_kernel<<<(int)std::min<int64_t>((P->n + 255) / 256, 2048), 256, 0, st>>>(
          P->n, ld, P->scal, P->cost.inv_scale, P->cost.norms, P->b, P->b_bar, P->beta);
  }
  if (!eval && !gram && !(flags & (LEANOT_SWEEP_ROWS_ONLY | LEANOT_SWEEP_COLS_ONLY)) &&
      ((flags & LEANOT_SWEEP_FUSED) || fused_default())) {
    const int rc = try_fused_sweep(*P, st);
    if (rc == LEANOT_OK) return check_launch("dxg_sweep(fused)");
    if (rc != LEANOT_EINVAL) return rc;
  }
  if (!eval && !gram && !(flags & (LEANOT_SWEEP_ROWS_ONLY | LEANOT_SWEEP_COLS_ONLY | LEANOT_SWEEP_TWO_PASS))) {
    const int rc = try_sr_sweep(*P, st, (flags & LEANOT_SWEEP_SINGLE_READ) != 0);
    if (rc == LEANOT_OK) return check_launch("dxg_sweep(single-read)");
    if (rc != LEANOT_EINVAL) return rc;
  }
  if (!(flags & LEANOT_SWEEP_COLS_ONLY)) LEANOT_TRY(launch_rowpass(A, 2, eval, st));
  if (flags & LEANOT_SWEEP_ROWS_ONLY) return check_launch("dxg_sweep(rows)");
  ColPassArgs B;
  memset(&B, 0, sizeof(B));
  B.cost = A.cost; B.i0 = P->row0; B.i1 = P->row1; B.a = P->scal;
  B.b[0] = A.b[0]; B.b[1] = A.b[1];
  B.m = P->m; B.coef = P->coef; B.slab = P->slab; B.splits = P->splits; B.gram = A.gram;
  LEANOT_TRY(launch_colpass(B, 2, st));
  LEANOT_TRY(launch_slab_reduce(P->slab, P->splits, 2, P->n, P->col, st));
  return check_launch("dxg_sweep");
}

int leanot_dxg_update(const leanot_dxg_plan_t* P, void* stream) {
  LEANOT_TRY(validate_plan(P));
  LEANOT_TRY(ensure_init());
  cudaStream_t st = S_(stream);
  UpdArgs U = make_upd(*P);
  if (small_plan(*P)) {
    // all O(n) updates in one CTA (the sweep already reduced the slabs into col)
    dxg_update_small<<<1, 1024, 0, st>>>(U);
    return check_launch("dxg_update_small");
  }
  dxg_update1<<<P->nblk_upd, 256, 0, st>>>(U);
  dxg_update2<<<P->nblk_upd, 256, 0, st>>>(U, 1);
  dxg_update3<<<P->nblk_upd, 256, 0, st>>>(U);
  return check_launch("dxg_update");
}

int leanot_dxg_eval(const leanot_dxg_plan_t* P, void* stream) {
  LEANOT_TRY(validate_plan(P));
  LEANOT_TRY(ensure_init());
  cudaStream_t st = S_(stream);
  if (use_sep(*P)) {
    LEANOT_TRY(sep_dxg_eval(*P, st));
    return check_launch("dxg_eval(separable)");
  }
  const int64_t nr = P->row1 - P->row0;
  const double* v = P->rowstat + 2 * nr;  // row minima (eta = 0 form)
  if (P->prm.eta > 0) {
    // LSE_j(-(C_ij + sd_j)/eta) with an exact max (dxg.py:337); the shift is -min_j(C_ij + sd_j)/eta
    // from the evaluation sweep's row minima (one read of C).  The LSEs go to S[nr, 2nr) (the
    // midpoint row sums, not read after the sweep), so the minima stay intact and a second
    // call gives the same result.
    double* L = P->S + nr;
    LEANOT_TRY(launch_rowlse(make_view(P->cost), P->row0, P->row1, P->sd, 1.0, -1.0 / P->prm.eta, L, st,
                             P->rowstat + 2 * nr));
    v = L;
  }
  rowstats_reduce_kernel<<<1, 1024, 0, st>>>(nr, P->row0, P->r, P->S, P->m, P->rowstat, v, P->evalbuf);
  colstats_reduce_kernel<<<1, 1024, 0, st>>>(P->n, P->col, P->c, P->delta, P->evalbuf + 3);
  return check_launch("dxg_eval");
}

int leanot_dxg_iterate(const leanot_dxg_plan_t* P, int iters, void* stream) {
  LEANOT_TRY(validate_plan(P));
  LEANOT_TRY(ensure_init());
  if (try_persist_iterate(*P, iters, S_(stream)) == LEANOT_OK) return check_launch("dxg_iterate(persistent)");
  for (int i = 0; i < iters; ++i) {
    LEANOT_TRY(leanot_dxg_sweep(P, 0, stream));
    LEANOT_TRY(leanot_dxg_update(P, stream));
  }
  return LEANOT_OK;
}

int leanot_dxg_iterate_eval(const leanot_dxg_plan_t* P, int iters, int start_update, void* stream) {
  LEANOT_TRY(validate_plan(P));
  LEANOT_TRY(ensure_init());
  g_err[0] = 0;
  const int rc = try_rowowner_iterate_eval(*P, iters, start_update, S_(stream));
  if (rc != LEANOT_OK) {
    if (!g_err[0]) set_error("dxg_iterate_eval: plan not eligible (single-process, n <= 1024, non-separable cost)");
    return rc;
  }
  return check_launch("dxg_iterate_eval");
}

int leanot_graph_create(const leanot_dxg_plan_t* P, int iters, void** graph_exec, void* stream) {
  LEANOT_TRY(validate_plan(P));
  LEANOT_TRY(ensure_init());
  cudaStream_t cap;
  if (cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess) { set_error("stream create"); return LEANOT_ECUDA; }
  // make sure lazy attribute setup happened outside capture
  {
    int rc = leanot_dxg_iterate(P, 0, stream);
    if (rc) return rc;
  }
  cudaGraph_t g;
  cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) { set_error("begin capture: %s", cudaGetErrorString(e)); cudaStreamDestroy(cap); return LEANOT_ECUDA; }
  int rc = leanot_dxg_iterate(P, iters, cap);
  e = cudaStreamEndCapture(cap, &g);
  cudaStreamDestroy(cap);
  if (rc != LEANOT_OK) return rc;
  if (e != cudaSuccess) { set_error("end capture: %s", cudaGetErrorString(e)); return LEANOT_ECUDA; }
  cudaGraphExec_t ex;
  e = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) { set_error("instantiate: %s", cudaGetErrorString(e)); return LEANOT_ECUDA; }
  *graph_exec = ex;
  (void)stream;
  return LEANOT_OK;
}

int leanot_graph_launch(void* graph_exec, void* stream) {
  cudaError_t e = cudaGraphLaunch(reinterpret_cast<cudaGraphExec_t>(graph_exec), S_(stream));
  if (e != cudaSuccess) { set_error("graph launch: %s", cudaGetErrorString(e)); return LEANOT_ECUDA; }
  return LEANOT_OK;
}

int leanot_graph_destroy(void* graph_exec) {
  if (graph_exec) cudaGraphExecDestroy(reinterpret_cast<cudaGraphExec_t>(graph_exec));
  return LEANOT_OK;
}

int leanot_bary_rmap(const double* L, int m, int64_t n, const double* w, double* r, double* scratch, void* stream) {
  LEANOT_TRY(ensure_init());
  if (m < 1 || m > LEANOT_MAX_K) { set_error("barycenter supports 1..16 marginals"); return LEANOT_EINVAL; }
  cudaStream_t st = S_(stream);
  launch_rmap(L, m, n, w, scratch, scratch + n, r, st);
  return check_launch("bary_rmap");
}

int leanot_sync(void* stream) {
  cudaError_t e = cudaStreamSynchronize(S_(stream));
  if (e != cudaSuccess) { set_error("sync: %s", cudaGetErrorString(e)); return LEANOT_ECUDA; }
  return LEANOT_OK;
}

}  // extern "C"
