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
//
// Two implementations of one LSE-convolution stage, chosen on device per table:
//  * linear domain on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64): with
//    M = max over the summed axis, Y = M + log(exp(X - M) . K), K[t][q] = exp(g[|q-t|]).
//    Valid while every finite g lies in [-600, 600] (K and the products stay normal
//    doubles; dropped terms are < e^-145 of the largest).  All terms are positive, so
//    the sum is accurate to a few ulps -- the same bar as the exact LSE.
//  * log domain (sep_axis_kernel): exact max-shifted LSE per output, any g.
// The table kernel writes a device flag `lin` that selects the path, so graph replays
// and device-resident scalars (a) need no host round trip.

namespace leanot {

// Y[p][q] = LSE_{q'} (X[p][q'] + g[|q-q'|])  (axis 1)   or   LSE_{p'} (X[p'][q] + g[|p-p'|])  (axis 0)
// MIN mode: min instead of LSE.  One thread per output; two passes (exact max, then the
// max-shifted sum with the table exp of leanot_common.cuh, zero integer shift).
template <bool MIN>
__global__ void __launch_bounds__(256) sep_axis_kernel(const double* __restrict__ X, const double* __restrict__ g,
                                                       int H, int W, int axis, double* __restrict__ Y,
                                                       const int* __restrict__ skip, int64_t xs, int64_t ys) {
  if (skip && *skip) return;  // the tensor-core path handles this table
  X += blockIdx.y * xs;       // batch of independent grids (blockIdx.y)
  Y += blockIdx.y * ys;
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

// K[t][q] = exp(g[|q - t|]) for t, q < L (row-major L x L).  Block 0 also writes lin:
// 1 if every finite g[d], d < D, lies in [-600, 600] (and allow != 0), else 0.
__global__ void sep_kmat_kernel(const double* __restrict__ g, int L, int D, int allow, double* __restrict__ K,
                                int* __restrict__ lin) {
  if (blockIdx.x == 0) {
    __shared__ int bad;
    if (threadIdx.x == 0) bad = allow ? 0 : 1;
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      const double v = g[d];
      if (v != v || (v != -INFINITY && (v < -600.0 || v > 600.0))) atomicOr(&bad, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) *lin = bad ? 0 : 1;
  }
  const int64_t total = (int64_t)L * L;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(e / L), q = (int)(e % L);
    K[e] = exp(g[abs(q - t)]);
  }
}

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// One LSE-convolution stage as an FP64 tensor-core GEMM with the exp fused into the operand
// load and the log into the epilogue (grid cells row-major, H x W):
//   AX = 1:  Y[p][q] = M[p] + log sum_t exp(X[p][t] - M[p]) K[t][q]      (K = K_W, W x W)
//   AX = 0:  Y[p][q] = M[q] + log sum_p' K[p][p'] exp(X[p'][q] - M[q])   (K = K_H, H x H)
// M = exact max over the summed axis, computed by each CTA for its 32 rows / columns.
// 32 x 32 output tile per CTA, 4 warps of 16 x 16 (2 x 2 DMMA m8n8k4), K staged 32 at a time
// with a register prefetch of the next stage; padded shared strides keep fragment loads at
// the minimum two wavefronts.
template <int AX>
__global__ void __launch_bounds__(128) sep_lse_gemm_kernel(const double* __restrict__ X, const double* __restrict__ K,
                                                           int H, int W, double* __restrict__ Y,
                                                           const int* __restrict__ lin, int64_t xs, int64_t ys) {
  if (!*lin) return;
  X += blockIdx.z * xs;  // batch of independent grids (blockIdx.z), one kernel matrix
  Y += blockIdx.z * ys;
  constexpr int BT = 32, BK = 32, S = BK + 4;
  __shared__ double As[2][BT * S];
  __shared__ double Bs[2][BK * S];
  __shared__ double Ms[BT];
  __shared__ double red[4][BT];
  const int Kd = AX == 1 ? W : H;
  const int m0 = blockIdx.y * BT, n0 = blockIdx.x * BT;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // exact max over the summed axis for this CTA's rows (AX = 1) or columns (AX = 0)
  if (AX == 1) {
    for (int rr = warp; rr < BT; rr += 4) {
      const int p = m0 + rr;
      double m = -INFINITY;
      if (p < H)
        for (int t = lane; t < W; t += 32) m = fmax(m, X[(int64_t)p * W + t]);
      m = warp_max(m);
      if (lane == 0) Ms[rr] = m;
    }
  } else {
    const int q = n0 + lane;
    double m = -INFINITY;
    if (q < W)
      for (int p = warp; p < H; p += 4) m = fmax(m, X[(int64_t)p * W + q]);
    red[warp][lane] = m;
    __syncthreads();
    if (warp == 0) Ms[lane] = fmax(fmax(red[0][lane], red[1][lane]), fmax(red[2][lane], red[3][lane]));
  }
  __syncthreads();
  // stage loader: each thread moves 8 A and 8 B elements (rows e/32, cols e%32 of the tiles)
  double ra[8], rb[8];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = tid + u * 128, r = e >> 5, c = e & 31;
      // A tile: rows m0 + r, k = k0 + c;  B tile: k = k0 + r, cols n0 + c
      const int ar = m0 + r, ak = k0 + c, bk = k0 + r, bc = n0 + c;
      if (AX == 1) {
        ra[u] = (ar < H && ak < Kd) ? X[(int64_t)ar * W + ak] : -INFINITY;
        rb[u] = (bk < Kd && bc < W) ? K[(int64_t)bk * W + bc] : 0.0;
      } else {
        ra[u] = (ar < H && ak < Kd) ? K[(int64_t)ar * H + ak] : 0.0;
        rb[u] = (bk < Kd && bc < W) ? X[(int64_t)bk * W + bc] : -INFINITY;
      }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = tid + u * 128, r = e >> 5, c = e & 31;
      double a = ra[u], b = rb[u];
      if (AX == 1) {
        const double m = Ms[r];
        a = (m == -INFINITY || a == -INFINITY) ? 0.0 : exp(a - m);
      } else {
        const double m = Ms[c];
        b = (m == -INFINITY || b == -INFINITY) ? 0.0 : exp(b - m);
      }
      As[buf][r * S + c] = a;
      Bs[buf][r * S + c] = b;
    }
  };
  const int wm = (warp >> 1) * 16, wn = (warp & 1) * 16;
  const int fr = lane >> 2, fc = lane & 3;
  double acc[2][2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  fetch(0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < Kd; k0 += BK) {
    const bool more = k0 + BK < Kd;
    if (more) fetch(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[2], bf[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = As[buf][(wm + i * 8 + fr) * S + kk + fc];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = Bs[buf][(kk + fc) * S + wn + j * 8 + fr];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int rl = wm + i * 8 + fr, row = m0 + rl;
    if (row >= H) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cl = wn + j * 8 + 2 * fc + h, col = n0 + cl;
        if (col >= W) continue;
        const double mv = AX == 1 ? Ms[rl] : Ms[cl];
        Y[(int64_t)row * W + col] = mv == -INFINITY ? -INFINITY : mv + log(acc[i][j][h]);
      }
  }
}

// elementwise helpers over nz batches of n cells (input batch stride is, output os)
#define SEP_EW_LOOP                                                                                  \
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)nz * n;             \
       e += (int64_t)gridDim.x * blockDim.x)
__global__ void sep_neg_kernel(const double* b, int64_t n, double* out, int nz = 1, int64_t is = 0,
                               int64_t os = 0) {  // out = -b
  SEP_EW_LOOP {
    const int64_t z = e / n, i = e - z * n;
    out[z * os + i] = -b[z * is + i];
  }
}
// log r - L (r shared by the batch, L batch stride is)
__global__ void sep_logw_kernel(const double* r, const double* L, int64_t n, double* out, int nz = 1, int64_t is = 0,
                                int64_t os = 0) {
  SEP_EW_LOOP {
    const int64_t z = e / n, i = e - z * n;
    out[z * os + i] = r[i] > 0 ? log(r[i]) - L[z * is + i] : -INFINITY;
  }
}
// col = exp(V - b): V batch stride n, b stride bs, col stride os
__global__ void sep_col_kernel(const double* V, const double* b, int64_t n, double* col, int nz = 1, int64_t bs = 0,
                               int64_t os = 0) {
  SEP_EW_LOOP {
    const int64_t z = e / n, i = e - z * n;
    col[z * os + i] = exp(V[z * n + i] - b[z * bs + i]);
  }
}
// log|b| - b (b <= 0 after recentering)
__global__ void sep_logabsb_kernel(const double* b, int64_t n, double* out, int nz = 1, int64_t is = 0,
                                   int64_t os = 0) {
  SEP_EW_LOOP {
    const int64_t z = e / n, i = e - z * n;
    const double v = b[z * is + i];
    out[z * os + i] = v != 0.0 ? log(fabs(v)) - v : -INFINITY;
  }
}
__global__ void sep_scale_kernel(const double* x, double sc, int64_t n, double* out, int nz = 1, int64_t is = 0,
                                 int64_t os = 0) {
  SEP_EW_LOOP {
    const int64_t z = e / n, i = e - z * n;
    out[z * os + i] = x[z * is + i] * sc;
  }
}
#undef SEP_EW_LOOP

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

static bool sep_gemm_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LEANOT_SEP_GEMM");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// one g table and, for the LSE modes, its linear-domain kernel matrices + path flag
struct SepTab {
  const double* g;
  const double* Kw;  // W x W
  const double* Kh;  // H x H
  const int* lin;    // device flag: 1 = tensor-core path
};

// scratch layout (doubles): 6 n-vectors, 4 tables of D, 64 spare, three (W^2 + H^2)
// kernel-matrix slots and the three path flags
static int64_t sep_ws_doubles(const leanot_cost_t& c) {
  const int64_t D = c.height > c.width ? c.height : c.width;
  const int64_t KM = (int64_t)c.width * c.width + (int64_t)c.height * c.height;
  return 6 * c.n + 4 * D + 3 * KM + 128;
}

struct SepCtx {
  int H, W, p;
  int64_t n;
  double inv;
  cudaStream_t st;
  int nb;
  double* K[3];
  int* lin;
  SepTab table(const double* a_ptr, int mode, double* g, double eta = 1.0) const {
    const int D = H > W ? H : W;
    sep_table_kernel<<<(D + 255) / 256, 256, 0, st>>>(a_ptr, p, inv, eta, D, mode, g);
    SepTab t{g, nullptr, nullptr, nullptr};
    if (mode == 2) return t;  // min-plus table: log domain only
    const int slot = mode == 0 ? 0 : (mode == 1 ? 1 : 2);
    double* Kw = K[slot];
    double* Kh = Kw + (int64_t)W * W;
    const int allow = sep_gemm_env() ? 1 : 0;
    sep_kmat_kernel<<<(int)std::min<int64_t>(((int64_t)W * W + 255) / 256, 1024), 256, 0, st>>>(g, W, D, allow, Kw,
                                                                                                lin + slot);
    sep_kmat_kernel<<<(int)std::min<int64_t>(((int64_t)H * H + 255) / 256, 1024), 256, 0, st>>>(g, H, D, allow, Kh,
                                                                                                lin + slot);
    t.Kw = Kw;
    t.Kh = Kh;
    t.lin = lin + slot;
    return t;
  }
  // Y = LSE-convolution of X along grid axis ax (1: within rows over W, 0: within columns over H)
  // nz independent grids: X + z*xs -> Y + z*ys (xs, ys default to n)
  void axis(const double* X, const SepTab& t, int ax, double* Y, int nz = 1, int64_t xs = -1, int64_t ys = -1) const {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(sep_axis_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TAB_BYTES);
      attr = true;
    }
    if (xs < 0) xs = n;
    if (ys < 0) ys = n;
    const dim3 gg((W + 31) / 32, (H + 31) / 32, nz);
    if (ax == 1) sep_lse_gemm_kernel<1><<<gg, 128, 0, st>>>(X, t.Kw, H, W, Y, t.lin, xs, ys);
    else sep_lse_gemm_kernel<0><<<gg, 128, 0, st>>>(X, t.Kh, H, W, Y, t.lin, xs, ys);
    sep_axis_kernel<false><<<dim3(nb, nz), 256, TAB_BYTES, st>>>(X, t.g, H, W, ax, Y, t.lin, xs, ys);
  }
  void axis_min(const double* X, const double* g, int ax, double* Y) const {
    sep_axis_kernel<true><<<nb, 256, 0, st>>>(X, g, H, W, ax, Y, nullptr, 0, 0);
  }
  int eg(int nz = 1) const { return (int)std::min<int64_t>((nz * n + 255) / 256, 4096); }
};

static SepCtx make_sep(const leanot_cost_t& c, cudaStream_t st, double* ws) {
  SepCtx s;
  s.H = c.height; s.W = c.width; s.p = c.p; s.n = c.n; s.inv = c.inv_scale; s.st = st;
  s.nb = (int)std::min<int64_t>((c.n + 255) / 256, (int64_t)num_sms() * 3);
  const int64_t D = c.height > c.width ? c.height : c.width;
  const int64_t KM = (int64_t)c.width * c.width + (int64_t)c.height * c.height;
  s.K[0] = ws + 6 * c.n + 4 * D + 64;
  s.K[1] = s.K[0] + KM;
  s.K[2] = s.K[1] + KM;
  s.lin = reinterpret_cast<int*>(s.K[2] + KM);
  return s;
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
  double* ws = P.slab;  // engine sizes the slab >= sep_ws_doubles for grid costs
  const SepCtx s = make_sep(P.cost, st, ws);
  const int64_t n = P.n;
  const int D = s.H > s.W ? s.H : s.W;
  double *T = ws, *L = ws + n, *U = ws + 2 * n, *V = ws + 3 * n, *X = ws + 4 * n, *Y = ws + 5 * n;
  double *g = ws + 6 * n, *g2 = g + D, *g3 = g2 + D, *g4 = g3 + D;
  const int eg = s.eg();
  for (int k = 0; k < 2; ++k) {
    const double* bk = k == 0 ? P.b : P.b_bar;
    const SepTab tg = s.table(P.scal + k, 0, g);
    sep_neg_kernel<<<eg, 256, 0, st>>>(bk, n, X);
    s.axis(X, tg, 1, T);
    s.axis(T, tg, 0, L);
    if (eval && k == 0) {
      // cost: log sum_j e^{x_ij} f(dr)/s  and  ... f(dc)/s
      const SepTab tg2 = s.table(P.scal, 1, g2);
      double* Cr = P.rowstat;           // nr
      double* Cc = P.rowstat + n;       // nr
      s.axis(T, tg2, 0, Cr);            // f(dr) weight on the row stage
      s.axis(X, tg2, 1, Y);             // f(dc) weight on the column stage
      s.axis(Y, tg, 0, Cc);
      // B = log sum_j e^{x_ij} |b_j|
      sep_logabsb_kernel<<<eg, 256, 0, st>>>(bk, n, Y);
      s.axis(Y, tg, 1, U);
      s.axis(U, tg, 0, V);
      double* Bl = P.bprime;            // scratch n-vector free during the sweep
      cudaMemcpyAsync(Bl, V, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
      // dual row reductions of C + sd (min-plus for eta = 0, LSE of -(C + sd)/eta otherwise)
      double* dv = P.rowstat + 2 * n;
      if (P.prm.eta > 0) {
        const SepTab tg3 = s.table(nullptr, 3, g3, P.prm.eta);
        sep_scale_kernel<<<eg, 256, 0, st>>>(P.sd, -1.0 / P.prm.eta, n, Y);
        s.axis(Y, tg3, 1, U);
        s.axis(U, tg3, 0, dv);
      } else {
        s.table(nullptr, 2, g4);
        s.axis_min(P.sd, g4, 1, U);
        s.axis_min(U, g4, 0, dv);
      }
      // keep L of weight set 0 for the reduce
      cudaMemcpyAsync(P.S, L, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
    }
    // column marginal with row weights r
    sep_logw_kernel<<<eg, 256, 0, st>>>(P.r, L, n, X);
    s.axis(X, tg, 1, U);
    s.axis(U, tg, 0, V);
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

// batched scratch of the barycenter plans: 4 (m x n) blocks after the separable layout
// (barycenter.py sizes the slab as leanot_grid_sep_ws_doubles + 4 m n)
struct BarySepWs {
  double *Xa, *Ta, *Ya, *Ua;
};
static BarySepWs bary_sep_ws(const leanot_bary_plan_t& P) {
  const int64_t mn = (int64_t)P.m * P.n;
  double* B = P.slab + sep_ws_doubles(P.cost);
  return {B, B + mn, B + 2 * mn, B + 3 * mn};
}

// all 2m row log-normalizers into P.L ([w][k][i]); eval: per-k stats of weight set 0.
// The m marginals of a weight set share the kernel table, so every stage runs as one
// batched launch over k.
static int sep_bary_rows(const leanot_bary_plan_t& P, bool eval, cudaStream_t st) {
  double* ws = P.slab;
  const SepCtx s = make_sep(P.cost, st, ws);
  const int64_t n = P.n, ns = P.ns;
  const int m = P.m;
  const int D = s.H > s.W ? s.H : s.W;
  const BarySepWs B = bary_sep_ws(P);
  double *g = ws + 6 * n, *g2 = g + D;
  const int eg = s.eg(m);
  for (int w = 0; w < 2; ++w) {
    const SepTab tg = s.table(P.scal + w, 0, g);
    const double* bw = w == 0 ? P.b : P.b_bar;
    double* Lw = P.L + (int64_t)w * m * n;
    sep_neg_kernel<<<eg, 256, 0, st>>>(bw, n, B.Xa, m, ns, n);
    s.axis(B.Xa, tg, 1, B.Ta, m);
    s.axis(B.Ta, tg, 0, Lw, m);
    if (eval && w == 0) {
      const SepTab tg2 = s.table(P.scal, 1, g2);
      s.axis(B.Ta, tg2, 0, P.rowstat, m, n, 3 * n);          // Cr_k
      s.axis(B.Xa, tg2, 1, B.Ya, m);
      s.axis(B.Ya, tg, 0, P.rowstat + n, m, n, 3 * n);       // Cc_k
      sep_logabsb_kernel<<<eg, 256, 0, st>>>(bw, n, B.Ya, m, ns, n);
      s.axis(B.Ya, tg, 1, B.Ua, m);
      s.axis(B.Ua, tg, 0, P.S + n, m, n, 2 * n);             // B_k (log sum e^x |b|)
      cudaMemcpy2DAsync(P.S, 2 * n * sizeof(double), Lw, n * sizeof(double), n * sizeof(double), m,
                        cudaMemcpyDeviceToDevice, st);        // L_k next to B_k
    }
  }
  return LEANOT_OK;
}

// column marginals of all (k, w) with row weights r_w (P.r, after the r-maps)
static int sep_bary_cols(const leanot_bary_plan_t& P, cudaStream_t st) {
  double* ws = P.slab;
  const SepCtx s = make_sep(P.cost, st, ws);
  const int64_t n = P.n, ns = P.ns;
  const int m = P.m;
  const BarySepWs B = bary_sep_ws(P);
  double* g = ws + 6 * n;
  const int eg = s.eg(m);
  for (int w = 0; w < 2; ++w) {
    const SepTab tg = s.table(P.scal + w, 0, g);
    const double* bw = w == 0 ? P.b : P.b_bar;
    sep_logw_kernel<<<eg, 256, 0, st>>>(P.r + w * n, P.L + (int64_t)w * m * n, n, B.Xa, m, n, n);
    s.axis(B.Xa, tg, 1, B.Ua, m);
    s.axis(B.Ua, tg, 0, B.Ta, m);
    sep_col_kernel<<<eg, 256, 0, st>>>(B.Ta, bw, n, P.col + w * n, m, ns, 2 * n);
  }
  return LEANOT_OK;
}

static int sep_bary_eval(const leanot_bary_plan_t& P, cudaStream_t st) {
  double* ws = P.slab;
  const SepCtx s = make_sep(P.cost, st, ws);
  const int64_t n = P.n, ns = P.ns;
  const int m = P.m;
  const int D = s.H > s.W ? s.H : s.W;
  const BarySepWs B = bary_sep_ws(P);
  double* zero = ws + 5 * n;
  double* g3 = ws + 6 * n + 2 * D;
  cudaMemsetAsync(zero, 0, n * sizeof(double), st);
  const SepTab tg3 = s.table(nullptr, 3, g3, P.prm.eta);
  for (int k = 0; k < m; ++k) {
    const double* Cr = P.rowstat + (int64_t)k * 3 * n;
    sep_rowstats_kernel<<<1, 1024, 0, st>>>(n, P.r, P.S + (int64_t)k * 2 * n, Cr, Cr + n,
                                            P.S + (int64_t)k * 2 * n + n, P.scal, zero, P.evalbuf + k * 4);
    colstats_reduce_kernel<<<1, 1024, 0, st>>>(n, P.col + (int64_t)k * 2 * n, P.c + k * ns, P.delta + k * ns,
                                               P.evalbuf + 64 + k * 2);
  }
  // log_z[k] = LSE_j(-(C_ij + sd_kj)/eta) (barycenter.py:186-191)
  sep_scale_kernel<<<s.eg(m), 256, 0, st>>>(P.sd, -1.0 / P.prm.eta, n, B.Ya, m, ns, n);
  s.axis(B.Ya, tg3, 1, B.Ua, m);
  s.axis(B.Ua, tg3, 0, P.L, m);
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
  const SepCtx s = make_sep(*cost, st, ws);
  const int64_t n = cost->n;
  double *T = ws, *X = ws + n, *g = ws + 6 * n;
  const SepTab tg = s.table(a_dev, 0, g);
  sep_neg_kernel<<<s.eg(), 256, 0, st>>>(b, n, X);
  s.axis(X, tg, 1, T);
  s.axis(T, tg, 0, L);
  return check_launch("grid_sep_lse");
}

int leanot_grid_sep_colsum(const leanot_cost_t* cost, const double* a_dev, const double* b, const double* logw,
                           double* col, double* ws, void* stream) {
  using namespace leanot;
  LEANOT_TRY(validate_cost(cost));
  if (cost->kind != LEANOT_COST_GRID) { set_error("separable path needs a grid cost"); return LEANOT_EINVAL; }
  LEANOT_TRY(ensure_init());
  cudaStream_t st = S_(stream);
  const SepCtx s = make_sep(*cost, st, ws);
  const int64_t n = cost->n;
  double *U = ws, *V = ws + n, *g = ws + 6 * n;
  const SepTab tg = s.table(a_dev, 0, g);
  s.axis(logw, tg, 1, U);
  s.axis(U, tg, 0, V);
  sep_col_kernel<<<s.eg(), 256, 0, st>>>(V, b, n, col);
  return check_launch("grid_sep_colsum");
}

}  // extern "C"
