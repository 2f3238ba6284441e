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

// Linear-domain operand of one LSE-convolution stage (batched over blockIdx.z, grid cells
// row-major H x W):  M = exact max over the summed axis, E = exp(X - M) (0 where M = -inf).
//   AX = 1: one warp per grid row p, M[p] = max_t X[p][t]
//   AX = 0: 32 grid columns x 32 row groups per block, M[q] = max_p X[p][q]
template <int AX>
__global__ void __launch_bounds__(1024) sep_maxexp_kernel(const double* __restrict__ X, int H, int W, int64_t xs,
                                                         double* __restrict__ E, double* __restrict__ M, int md,
                                                         const int* __restrict__ lin) {
  if (!*lin) return;
  const int64_t n = (int64_t)H * W;
  X += blockIdx.z * xs;
  E += blockIdx.z * n;
  M += (int64_t)blockIdx.z * md;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (AX == 1) {
    const int p = blockIdx.x * 8 + warp;
    if (p >= H) return;
    const double* x = X + (int64_t)p * W;
    double m = -INFINITY;
    for (int t = lane; t < W; t += 32) m = fmax(m, x[t]);
    m = warp_max(m);
    double* e = E + (int64_t)p * W;
    for (int t = lane; t < W; t += 32) e[t] = m == -INFINITY ? 0.0 : exp(x[t] - m);
    if (lane == 0) M[p] = m;
  } else {
    // 32 columns x (blockDim / 32) row groups
    __shared__ double part[32][33];
    const int ng = blockDim.x >> 5;
    const int q = blockIdx.x * 32 + lane;
    double m = -INFINITY;
    if (q < W)
      for (int p = warp; p < H; p += ng) m = fmax(m, X[(int64_t)p * W + q]);
    part[warp][lane] = m;
    __syncthreads();
    m = part[0][lane];
    for (int g = 1; g < ng; ++g) m = fmax(m, part[g][lane]);
    if (q < W) {
      for (int p = warp; p < H; p += ng) {
        const int64_t o = (int64_t)p * W + q;
        E[o] = m == -INFINITY ? 0.0 : exp(X[o] - m);
      }
      if (warp == 0) M[q] = m;
    }
  }
}

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool ok) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
}

// Y = Mv + log(A . B) on the FP64 tensor cores, batched over blockIdx.z; row-major
// A (Mr x Kd), B (Kd x Nc), Y (Mr x Nc).  AX = 1: A = E_z, B = K_W, Mv_z indexed by row;
// AX = 0: A = K_H, B = E_z, Mv_z indexed by column.  BT x BT output tile per CTA, 4 warps
// of BT/2 x BT/2 (DMMA m8n8k4 tiles), K staged BK at a time through a 2-stage cp.async
// ring; padded shared strides keep the fragment loads at the minimum two wavefronts.
// BT = 32 for grids up to ~512 per side (enough CTAs to fill 148 SMs), 64 above.
template <int AX, int BT>
__global__ void __launch_bounds__(128) sep_gemm_log_kernel(const double* __restrict__ A, const double* __restrict__ B,
                                                           const double* __restrict__ Mv, int md, int Mr, int Nc,
                                                           int Kd, double* __restrict__ Y, int64_t ys,
                                                           const int* __restrict__ lin) {
  if (!*lin) return;
  constexpr int BK = BT == 32 ? 32 : 16, SA = BK + 4, SB = BT + 4;
  constexpr int WT = BT / 2, TI = WT / 8;  // warp tile, DMMA tiles per warp side
  constexpr int LA = BT * BK / 128;         // cp.async per thread per stage and operand
  __shared__ __align__(16) double As[2][BT * SA];
  __shared__ __align__(16) double Bs[2][BK * SB];
  const int64_t eo = (int64_t)blockIdx.z * Mr * Nc;  // E operand batch offset (H x W)
  if (AX == 1) A += eo; else B += eo;
  Mv += (int64_t)blockIdx.z * md;
  Y += blockIdx.z * ys;
  const int m0 = blockIdx.y * BT, n0 = blockIdx.x * BT;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = (warp >> 1) * WT, wn = (warp & 1) * WT;
  const int fr = lane >> 2, fc = lane & 3;
  auto stage = [&](int buf, int k0) {
#pragma unroll
    for (int u = 0; u < LA; ++u) {
      const int e = tid + u * 128;
      {
        const int r = e / BK, c = e % BK, gr = m0 + r, gk = k0 + c;
        const bool ok = gr < Mr && gk < Kd;
        cp_async8(&As[buf][r * SA + c], A + (ok ? (int64_t)gr * Kd + gk : 0), ok);
      }
      {
        const int r = e / BT, c = e % BT, gk = k0 + r, gc = n0 + c;
        const bool ok = gk < Kd && gc < Nc;
        cp_async8(&Bs[buf][r * SB + c], B + (ok ? (int64_t)gk * Nc + gc : 0), ok);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[TI][TI][2];
#pragma unroll
  for (int i = 0; i < TI; ++i)
#pragma unroll
    for (int j = 0; j < TI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nk = (Kd + BK - 1) / BK;
  stage(0, 0);
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) {
      stage(buf ^ 1, (kt + 1) * BK);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[TI], bf[TI];
#pragma unroll
      for (int i = 0; i < TI; ++i) af[i] = As[buf][(wm + i * 8 + fr) * SA + kk + fc];
#pragma unroll
      for (int j = 0; j < TI; ++j) bf[j] = Bs[buf][(kk + fc) * SB + wn + j * 8 + fr];
#pragma unroll
      for (int i = 0; i < TI; ++i)
#pragma unroll
        for (int j = 0; j < TI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TI; ++i) {
    const int row = m0 + wm + i * 8 + fr;
    if (row >= Mr) continue;
#pragma unroll
    for (int j = 0; j < TI; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn + j * 8 + 2 * fc + h;
        if (col >= Nc) continue;
        const double mv = AX == 1 ? Mv[row] : Mv[col];
        Y[(int64_t)row * Nc + col] = mv == -INFINITY ? -INFINITY : mv + log(acc[i][j][h]);
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
// kernel-matrix slots, the three path flags (2 doubles), then E (n) and Mv (D) for
// single-grid stages (batched barycenter stages place E / Mv in their own region)
static int64_t sep_ws_doubles(const leanot_cost_t& c) {
  const int64_t D = c.height > c.width ? c.height : c.width;
  const int64_t KM = (int64_t)c.width * c.width + (int64_t)c.height * c.height;
  return 6 * c.n + 4 * D + 3 * KM + 64 + 2 + c.n + D + 64;
}

struct SepCtx {
  int H, W, p;
  int64_t n;
  double inv;
  cudaStream_t st;
  int nb;
  double* K[3];
  double* E;   // linear-domain operand, batch x n
  double* Mv;  // its maxima, batch x max(H, W)
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
    const int md = H > W ? H : W;
    const bool small = (int64_t)((W + 63) / 64) * ((H + 63) / 64) * nz < 2 * (int64_t)num_sms();
    const int bt = small ? 32 : 64;
    const dim3 gg((W + bt - 1) / bt, (H + bt - 1) / bt, nz);
    if (ax == 1) {
      sep_maxexp_kernel<1><<<dim3((H + 7) / 8, 1, nz), 256, 0, st>>>(X, H, W, xs, E, Mv, md, t.lin);
      if (small) sep_gemm_log_kernel<1, 32><<<gg, 128, 0, st>>>(E, t.Kw, Mv, md, H, W, W, Y, ys, t.lin);
      else sep_gemm_log_kernel<1, 64><<<gg, 128, 0, st>>>(E, t.Kw, Mv, md, H, W, W, Y, ys, t.lin);
    } else {
      sep_maxexp_kernel<0><<<dim3((W + 31) / 32, 1, nz), 1024, 0, st>>>(X, H, W, xs, E, Mv, md, t.lin);
      if (small) sep_gemm_log_kernel<0, 32><<<gg, 128, 0, st>>>(t.Kh, E, Mv, md, H, W, H, Y, ys, t.lin);
      else sep_gemm_log_kernel<0, 64><<<gg, 128, 0, st>>>(t.Kh, E, Mv, md, H, W, H, Y, ys, t.lin);
    }
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
  s.E = s.K[2] + KM + 2;
  s.Mv = s.E + c.n;
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
  // single-process plans only: row-sharded (multi-GPU) barycenters take the dense sweeps
  return P.cost.kind == LEANOT_COST_GRID && P.row0 == 0 && P.row1 == P.n && sep_enabled_env();
}

// batched scratch of the barycenter plans: 4 (m x n) blocks after the separable layout
// (barycenter.py sizes the slab as leanot_grid_sep_ws_doubles + 4 m n)
struct BarySepWs {
  double *Xa, *Ta, *Ya, *Ua, *E, *Mv;
};
// (barycenter.py sizes the slab as leanot_grid_sep_ws_doubles + 5 m n + m max(H, W))
static BarySepWs bary_sep_ws(const leanot_bary_plan_t& P) {
  const int64_t mn = (int64_t)P.m * P.n;
  double* B = P.slab + sep_ws_doubles(P.cost);
  return {B, B + mn, B + 2 * mn, B + 3 * mn, B + 4 * mn, B + 5 * mn};
}

// all 2m row log-normalizers into P.L ([w][k][i]); eval: per-k stats of weight set 0.
// The m marginals of a weight set share the kernel table, so every stage runs as one
// batched launch over k.
static int sep_bary_rows(const leanot_bary_plan_t& P, bool eval, cudaStream_t st) {
  double* ws = P.slab;
  const BarySepWs B = bary_sep_ws(P);
  SepCtx s = make_sep(P.cost, st, ws);
  s.E = B.E;
  s.Mv = B.Mv;
  const int64_t n = P.n, ns = P.ns;
  const int m = P.m;
  const int D = s.H > s.W ? s.H : s.W;
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
  const BarySepWs B = bary_sep_ws(P);
  SepCtx s = make_sep(P.cost, st, ws);
  s.E = B.E;
  s.Mv = B.Mv;
  const int64_t n = P.n, ns = P.ns;
  const int m = P.m;
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
  const BarySepWs B = bary_sep_ws(P);
  SepCtx s = make_sep(P.cost, st, ws);
  s.E = B.E;
  s.Mv = B.Mv;
  const int64_t n = P.n, ns = P.ns;
  const int m = P.m;
  const int D = s.H > s.W ? s.H : s.W;
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

// Sinkhorn / IBP LSE on a grid, for nz potentials at once (IBP: one per marginal):
//   out_z,i = LSE_j((v_z,j - C_ij)/eta)    (sinkhorn.py:47-71)
// C is symmetric, so the same call gives the column LSEs of (phi_i - C_ij)/eta.
int64_t leanot_grid_sep_lse_eta_ws_doubles(const leanot_cost_t* cost, int nz) {
  const int64_t D = cost->height > cost->width ? cost->height : cost->width;
  return leanot::sep_ws_doubles(*cost) + (int64_t)nz * (3 * cost->n + D);
}

int leanot_grid_sep_lse_eta(const leanot_cost_t* cost, const double* v, int nz, int64_t vstride, double eta,
                            double* out, int64_t ostride, double* ws, void* stream) {
  using namespace leanot;
  LEANOT_TRY(validate_cost(cost));
  if (cost->kind != LEANOT_COST_GRID) { set_error("separable path needs a grid cost"); return LEANOT_EINVAL; }
  if (!(eta > 0)) { set_error("eta must be positive"); return LEANOT_EINVAL; }
  if (nz < 1 || vstride < cost->n || ostride < cost->n) { set_error("bad batch layout"); return LEANOT_EINVAL; }
  LEANOT_TRY(ensure_init());
  cudaStream_t st = S_(stream);
  SepCtx s = make_sep(*cost, st, ws);
  const int64_t n = cost->n;
  const int D = s.H > s.W ? s.H : s.W;
  double* B = ws + sep_ws_doubles(*cost);
  double *X = B, *T = B + nz * n;
  s.E = B + 2 * nz * n;
  s.Mv = B + 3 * nz * n;
  double* g3 = ws + 6 * n + 2 * D;
  const SepTab tg = s.table(nullptr, 3, g3, eta);          // g(d) = -f(d) inv / eta
  sep_scale_kernel<<<s.eg(nz), 256, 0, st>>>(v, 1.0 / eta, n, X, nz, vstride, n);
  s.axis(X, tg, 1, T, nz);
  s.axis(T, tg, 0, out, nz, n, ostride);
  return check_launch("grid_sep_lse_eta");
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
