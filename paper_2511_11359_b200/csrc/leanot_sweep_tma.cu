// TMA-staged sweeps for the stored cost (ExplicitKernel / HashKernel in HBM).
//
// Same arithmetic as rowpass_kernel / colpass_kernel, but C (and the column
// log-weights of pass A) stream into a shared-memory ring through 1-D bulk copies
// (cp.async.bulk ... mbarrier::complete_tx) issued by a dedicated producer warp, so
// the 16 consumer warps never wait on HBM latency and hold no prefetch registers.
//   pass A: stage = R rows x 960 columns of C + 960 columns of b and b_bar (45 KB), 3 stages
//   pass B: stage = 2 rows x 1920 columns of C (30 KB), 4 stages; 4 columns per thread
// Ring protocol: full[s] (1 producer arrival + tx bytes) / empty[s] (one arrival per
// consumer warp); phase parity = (step / NS) & 1.
// Included by leanot_lib.cu (single translation unit).

namespace leanot {

// 15 consumer warps + 1 producer warp = 512 threads, so ptxas grants 128 registers
// (a 17-warp CTA is rounded up to 20 warps for allocation and capped at 96).
constexpr int TP_THREADS = 480;          // consumer threads
constexpr int TP_ALL = TP_THREADS + 32;  // + producer warp

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void release_u32(uint32_t bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// a warp releases a stage once all its lanes are done reading it (one arrival per warp)
__device__ __forceinline__ void release(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(TP_THREADS) : "memory"); }

template <int K, int R, bool EVAL>
__global__ void __launch_bounds__(TP_ALL, 1) rowpass_tma_kernel(const RowPassArgs A) {
  constexpr int CH = 2 * TP_THREADS;   // columns per step
  constexpr int NS = 3;
  constexpr int STAGE = (R + K) * CH * 8;
  constexpr int NV = R * K + (EVAL ? 3 * R : 0);
  constexpr int NW = TP_THREADS / 32;
  extern __shared__ __align__(128) char smem[];
  char* stages = smem + TAB_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + NS * STAGE);
  uint64_t* empty = full + NS;
  double* red = reinterpret_cast<double*>(empty + NS);  // [NW][NV]
  load_table(reinterpret_cast<double*>(smem));
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, TP_THREADS / 32); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const CostView& cv = A.cost;
  const int64_t n = cv.n, nr = A.i1 - A.i0;
  const int64_t nblk = (nr + R - 1) / R, nch = (n + CH - 1) / CH;

  if (threadIdx.x >= TP_THREADS) {  // ---- producer warp ----
    if (threadIdx.x == TP_THREADS) {
      uint32_t q = 0;
      for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int64_t ib = A.i0 + blk * R;
        for (int64_t ch = 0; ch < nch; ++ch, ++q) {
          const int s = q % NS;
          mbar_wait(empty + s, ((q / NS) & 1) ^ 1);
          const int64_t j0 = ch * CH;
          const uint32_t w = (uint32_t)((n - j0 < CH ? n - j0 : CH) * 8);
          mbar_arrive_tx(full + s, (R + K) * w);
          char* dst = stages + s * STAGE;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int64_t i = ib + r < A.i1 ? ib + r : A.i1 - 1;
            bulk_g2s(dst + r * CH * 8, cv.mat + (i - cv.row_base) * cv.ld + j0, w, full + s);
          }
#pragma unroll
          for (int k = 0; k < K; ++k) bulk_g2s(dst + (R + k) * CH * 8, A.b[k] + j0, w, full + s);
        }
      }
    }
    return;
  }

  // ---- consumers ----
  const uint32_t tb = lane_tab_addr(smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double na[K];
#pragma unroll
  for (int k = 0; k < K; ++k) na[k] = -A.a[k];
  // ring position, kept incrementally (no division by NS, 32-bit counters) so the
  // per-stage bookkeeping stays small next to the 16 exps a thread does per stage
  uint32_t s = 0, ph = 0;
  const uint32_t full_u = smem_u32(full), empty_u = smem_u32(empty);
  const char* const st_base = stages + 16 * threadIdx.x;
  const int n32 = (int)n, nch32 = (int)nch;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t ib = A.i0 + blk * R;
    uint32_t mlo[R][K];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t i = ib + r < A.i1 ? ib + r : A.i1 - 1;
#pragma unroll
      for (int k = 0; k < K; ++k) mlo[r][k] = (uint32_t)shift_at(A, k, i - A.i0);
    }
    double acc[R][K], U[R], V[R], mn[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      U[r] = 0.0; V[r] = 0.0; mn[r] = INFINITY;
#pragma unroll
      for (int k = 0; k < K; ++k) acc[r][k] = 0.0;
    }
    int j = 2 * threadIdx.x;
#pragma unroll 2
    for (int ch = 0; ch < nch32; ++ch, j += CH) {
      mbar_wait_u32(full_u + 8 * s, ph);
      if (j < n32) {
        const char* st = st_base + s * STAGE;
        double2 bv[K];
#pragma unroll
        for (int k = 0; k < K; ++k) bv[k] = *reinterpret_cast<const double2*>(st + (R + k) * CH * 8);
        double2 sdv = make_double2(0.0, 0.0);
        if (EVAL) sdv = __ldg(reinterpret_cast<const double2*>(A.sd + j));
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double2 cc = *reinterpret_cast<const double2*>(st + r * CH * 8);
          const double c0 = cc.x, c1 = cc.y;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const double x0 = fma(na[k], c0, -bv[k].x);
            const double x1 = fma(na[k], c1, -bv[k].y);
            if (EVAL && k == 0) {
              const double e0 = texp(tb, x0, mlo[r][0]);
              const double e1 = texp(tb, x1, mlo[r][0]);
              acc[r][0] += e0 + e1;
              U[r] = fma(e0, c0, fma(e1, c1, U[r]));
              V[r] = fma(e0, x0, fma(e1, x1, V[r]));
              mn[r] = fmin(mn[r], fmin(c0 + sdv.x, c1 + sdv.y));
            } else {
              texp_acc(tb, x0, mlo[r][k], acc[r][k]);
              texp_acc(tb, x1, mlo[r][k], acc[r][k]);
            }
          }
        }
      }
      release_u32(empty_u + 8 * s);
      if (++s == NS) { s = 0; ph ^= 1; }
    }
    // block reduction over the consumer warps, fixed order
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const double v = warp_sum(acc[r][k]);
        if (lane == 0) red[warp * NV + r * K + k] = v;
      }
      if (EVAL) {
        const double u = warp_sum(U[r]), vv = warp_sum(V[r]), m = warp_min(mn[r]);
        if (lane == 0) {
          red[warp * NV + R * K + 3 * r] = u;
          red[warp * NV + R * K + 3 * r + 1] = vv;
          red[warp * NV + R * K + 3 * r + 2] = m;
        }
      }
    }
    consumer_sync();
    if (threadIdx.x < NV) {
      const int v = threadIdx.x;
      const bool is_min = EVAL && v >= R * K && ((v - R * K) % 3 == 2);
      double t = red[v];
      for (int w = 1; w < NW; ++w) t = is_min ? fmin(t, red[w * NV + v]) : t + red[w * NV + v];
      if (v < R * K) {
        const int r = v / K, k = v % K;
        const int64_t i = ib + r;
        if (i < A.i1) {
          const int64_t m = shift_at(A, k, i - A.i0);
          finalize_row(A, k, i - A.i0, t, m, m);
        }
      } else if (EVAL) {
        const int qq = v - R * K, r = qq / 3, s2 = qq % 3;
        const int64_t i = ib + r;
        if (i < A.i1) A.rowstat[s2 * nr + (i - A.i0)] = t;
      }
    }
    consumer_sync();
  }
}

// pass B, stored cost: 1920-column tiles x row splits, Q=2 rows per stage, 4 columns per
// thread as 2 column pairs at 2t and 2t + 960 (conflict-free 16-byte shared loads)
template <int K>
__global__ void __launch_bounds__(TP_ALL, 1) colpass_tma_kernel(const ColPassArgs A) {
  constexpr int V = 4;
  constexpr int TILE = V * TP_THREADS;  // 1920
  constexpr int PS = TILE / 2;          // pair stride
  constexpr int Q = 2;                  // rows per stage
  constexpr int NS = 4;
  constexpr int STAGE = Q * TILE * 8;   // 30 KB
  constexpr int CHUNK = 128;            // rows of per-row constants staged at once (CHUNK % Q == 0)
  extern __shared__ __align__(128) char smem[];
  char* stages = smem + TAB_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + NS * STAGE);
  uint64_t* empty = full + NS;
  double* s_coef = reinterpret_cast<double*>(empty + NS);              // [CHUNK][K][4]
  uint32_t* s_m = reinterpret_cast<uint32_t*>(s_coef + CHUNK * K * 4);  // [CHUNK][K]
  load_table(reinterpret_cast<double*>(smem));
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, TP_THREADS / 32); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const CostView& cv = A.cost;
  const int64_t n = cv.n, nr = A.i1 - A.i0;
  const int64_t ntiles = (n + TILE - 1) / TILE;
  const int64_t items = ntiles * A.splits;
  const int64_t rps = (nr + A.splits - 1) / A.splits;

  if (threadIdx.x >= TP_THREADS) {  // ---- producer warp ----
    if (threadIdx.x == TP_THREADS) {
      uint32_t q = 0;
      for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const int64_t tile = it % ntiles, split = it / ntiles;
        const int64_t j0 = tile * TILE;
        const uint32_t w = (uint32_t)((n - j0 < TILE ? n - j0 : TILE) * 8);
        const int64_t rs0 = A.i0 + split * rps;
        const int64_t rs1 = A.i1 < rs0 + rps ? A.i1 : rs0 + rps;
        // stage boundaries follow the consumers' chunks: CHUNK rows, Q rows per stage
        for (int64_t c0 = rs0; c0 < rs1; c0 += CHUNK) {
          const int64_t c1 = rs1 < c0 + CHUNK ? rs1 : c0 + CHUNK;
          for (int64_t r0 = c0; r0 < c1; r0 += Q, ++q) {
            const int s = q % NS;
            mbar_wait(empty + s, ((q / NS) & 1) ^ 1);
            const int nq = (int)(c1 - r0 < Q ? c1 - r0 : Q);
            mbar_arrive_tx(full + s, nq * w);
            for (int r = 0; r < nq; ++r)
              bulk_g2s(stages + s * STAGE + r * TILE * 8, cv.mat + (r0 + r - cv.row_base) * cv.ld + j0, w, full + s);
          }
        }
      }
    }
    return;
  }

  // ---- consumers ----
  const uint32_t tb = lane_tab_addr(smem);
  double na[K];
#pragma unroll
  for (int k = 0; k < K; ++k) na[k] = -A.a[k];
  uint32_t q = 0;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t tile = it % ntiles, split = it / ntiles;
    const int64_t nloc = n - tile * TILE;  // valid columns of this tile
    const int l0 = 2 * (int)threadIdx.x;
    const bool all_ok = l0 + PS + 1 < nloc;
    double nb[K][V], acc[K][V];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int lc = l0 + (v >> 1) * PS + (v & 1);
        nb[k][v] = lc < nloc ? -__ldg(A.b[k] + tile * TILE + lc) : 0.0;
        acc[k][v] = 0.0;
      }
    const int64_t rs0 = A.i0 + split * rps;
    const int64_t rs1 = A.i1 < rs0 + rps ? A.i1 : rs0 + rps;
    for (int64_t c0 = rs0; c0 < rs1; c0 += CHUNK) {
      const int nc = (int)(rs1 - c0 < CHUNK ? rs1 - c0 : CHUNK);
      consumer_sync();
      for (int t = threadIdx.x; t < nc * K * 4; t += TP_THREADS) {
        const int qq = t / (K * 4), k = (t / 4) % K, c = t % 4;
        s_coef[t] = A.coef[(k * nr + (c0 - A.i0 + qq)) * 4 + c];
      }
      for (int t = threadIdx.x; t < nc * K; t += TP_THREADS) {
        const int qq = t / K, k = t % K;
        s_m[t] = (uint32_t)A.m[k * nr + (c0 - A.i0 + qq)];
      }
      consumer_sync();
      for (int base = 0; base < nc; base += Q, ++q) {
        const int s = q % NS;
        mbar_wait(full + s, (q / NS) & 1);
        const int nq = nc - base < Q ? nc - base : Q;
        if (all_ok && nq == Q) {
          double c[Q][V];
#pragma unroll
          for (int r = 0; r < Q; ++r) {
            const char* rowp = stages + s * STAGE + r * TILE * 8 + 16 * threadIdx.x;
            const double2 ca = *reinterpret_cast<const double2*>(rowp);
            const double2 cb = *reinterpret_cast<const double2*>(rowp + PS * 8);
            c[r][0] = ca.x; c[r][1] = ca.y; c[r][2] = cb.x; c[r][3] = cb.y;
          }
#pragma unroll
          for (int r = 0; r < Q; ++r) {
            const int qq = base + r;
#pragma unroll
            for (int k = 0; k < K; ++k) {
              const double2 g01 = *reinterpret_cast<const double2*>(s_coef + (qq * K + k) * 4);
              const double2 g23 = *reinterpret_cast<const double2*>(s_coef + (qq * K + k) * 4 + 2);
              const uint32_t mlo = s_m[qq * K + k];
#pragma unroll
              for (int v = 0; v < V; ++v)
                texp_gacc(tb, fma(na[k], c[r][v], nb[k][v]), mlo, g01.x, g01.y, g23.x, g23.y, acc[k][v]);
            }
          }
        } else {
          for (int r = 0; r < nq; ++r) {
            const double* row = reinterpret_cast<const double*>(stages + s * STAGE + r * TILE * 8);
            const int qq = base + r;
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const int lc = l0 + (v >> 1) * PS + (v & 1);
              if (lc < nloc) {
                const double cv2 = row[lc];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                  const double* cf = s_coef + (qq * K + k) * 4;
                  texp_gacc(tb, fma(na[k], cv2, nb[k][v]), s_m[qq * K + k], cf[0], cf[1], cf[2], cf[3], acc[k][v]);
                }
              }
            }
          }
        }
        release(empty + s);
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double* out = A.slab + (split * K + k) * n + tile * TILE;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int lc = l0 + (v >> 1) * PS + (v & 1);
        if (lc < nloc) out[lc] = acc[k][v];
      }
    }
  }
}

template <int K, int R, bool EVAL>
static int launch_rowpass_tma_t(const RowPassArgs& A, cudaStream_t st) {
  constexpr int NV = R * K + (EVAL ? 3 * R : 0);
  const int smem = TAB_BYTES + 3 * (R + K) * 2 * TP_THREADS * 8 + 6 * 8 + (TP_THREADS / 32) * NV * 8;
  auto kern = rowpass_tma_kernel<K, R, EVAL>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return LEANOT_ECUDA;
    attr = true;
  }
  const int64_t nblk = (A.i1 - A.i0 + R - 1) / R;
  const int grid = (int)std::min<int64_t>(nblk, num_sms());
  if (grid < 1) return LEANOT_OK;
  kern<<<grid, TP_ALL, smem, st>>>(A);
  return LEANOT_OK;
}

template <int K>
static int launch_colpass_tma_t(const ColPassArgs& A, cudaStream_t st) {
  const int smem = TAB_BYTES + 4 * 2 * 4 * TP_THREADS * 8 + 8 * 8 + 128 * K * 4 * 8 + 128 * K * 4;
  auto kern = colpass_tma_kernel<K>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return LEANOT_ECUDA;
    attr = true;
  }
  const int64_t items = ((A.cost.n + 4 * TP_THREADS - 1) / (4 * TP_THREADS)) * A.splits;
  const int grid = (int)std::min<int64_t>(items, num_sms());
  if (grid < 1) return LEANOT_OK;
  kern<<<grid, TP_ALL, smem, st>>>(A);
  return LEANOT_OK;
}

// TMA path: stored cost, even n (16-byte bulk granularity), 16-byte aligned rows
static bool tma_ok(const CostView& cv) {
  return cv.kind == LEANOT_COST_STORED && (cv.n % 2) == 0 && (cv.ld % 2) == 0 && tma_enabled();
}

}  // namespace leanot
