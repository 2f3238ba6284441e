// Fused DXG sweep for the stored cost: pass A (row normalizers) and pass B (column
// sums) of one iteration in ONE persistent launch, with pass B trailing pass A by one
// row panel so that pass B's reads of C are served by L2 instead of HBM.
//
// Why: the two-pass sweep reads C (80 GB at n = 1e5) twice per iteration and runs at
// the board's 1 kW power cap; a DRAM byte costs ~60 pJ more than an L2 byte
// (profiles/r01_power.md), and pass A/B over L2-resident rows ran 21 %/14 % faster
// than over HBM in the same power envelope (profiles/r01_l2_reuse.md).  One HBM read
// per iteration is the minimum: a row must be normalized before any of its column
// contributions can be accumulated (dxg.py:199-203), and a row of C does not fit on
// chip, so pass B re-reads it -- from L2, one panel (16 rows, 12.8 MB) behind pass A.
//
// Schedule (G CTAs, one per SM, co-resident: cooperative launch):
//   CTA c owns the column tile [c W, (c+1) W) for the whole launch (its column sums stay
//   in registers: no slabs, no second-stage reduce) and one pass-A unit per panel:
//   R = 4 rows x one of Q column segments (P/R x Q = G units per panel).
//   step s: A(panel s): row partial sums of its unit -> part[s % NSLOT]; arrive cnt[s].
//           B(panel s-LAG): wait cnt[s-LAG] == units (normally set long before: every
//           CTA has done A(s-LAG) and 2 LAG - 1 phases since), S_i = sum over segments in
//           fixed order, g_i = r_i / S_i, then the tile's column sums over the panel.
//   A lag of 2 panels (~40 MB of C in flight at n = 1e5) keeps the re-reads in L2 while
//   absorbing the CTAs' step-to-step jitter (a lag of 1 stalled on the arrival counters).
//   C streams through one shared-memory ring (cp.async.bulk + mbarriers) fed by a
//   producer warp in exactly the consumers' order (A stages, then B stages).
// Arithmetic per element and weight set is that of rowpass/colpass (table exp with the
// previous iteration's row shift); rows whose sum leaves [2^-900, 2^900] are skipped by
// pass B and recomputed exactly afterwards (fused_fix_kernel), in ascending row order.
// Deterministic: fixed reduction orders, no floating-point atomics.
// Included by leanot_lib.cu after leanot_sweep_tma.cu (mbarrier / bulk-copy helpers).

namespace leanot {

constexpr int FU_CW = 11;                          // consumer warps
constexpr int FU_THREADS = FU_CW * 32;             // 352 consumer threads
constexpr int FU_PROD = FU_THREADS;                // producer warp (lane 0 issues the bulk copies)
constexpr int FU_COORD = FU_THREADS + 32;          // coordinator warp (arrivals, row constants)
constexpr int FU_ALL = FU_THREADS + 64;
constexpr int FU_R = 4;                            // rows per pass-A unit
constexpr int FU_P = 16;                           // rows per panel
constexpr int FU_RB = 4;                           // rows per pass-B stage
constexpr int FU_CHA = 2 * FU_THREADS;             // 704 columns per pass-A stage
constexpr int FU_NS = 4;                           // ring slots
constexpr int FU_SLOT = (FU_R + 2) * FU_CHA * 8;   // 33,792 B: A stage (4 rows + b, b_bar)
constexpr int FU_WMAX = FU_SLOT / (FU_RB * 8);     // max column tile (1056) of a B stage
constexpr int FU_LAG = 2;                          // pass B trails pass A by this many panels
constexpr int FU_NSLOT = 8;                        // panels of partial sums in flight (>= 2 LAG + 2)
// per-panel row constants, double-buffered: coef [P][2][4] doubles, shift [P][2] u32, ok [P][2] + 1 int
constexpr int FU_CBUF = (FU_P * 2 * 4 * 8 + FU_P * 2 * 4 + (FU_P * 2 + 2) * 4 + 15) & ~15;  // 16-byte multiple
constexpr int FU_NBAR = 16;                        // mbarrier words (2 NS + 5 used; keeps 16-byte alignment)
constexpr int FU_SMEM = TAB_BYTES + FU_NS * FU_SLOT + FU_NBAR * 8 + FU_CW * FU_R * 2 * 8 + 2 * FU_CBUF;
static_assert(2 * FU_NS + 5 <= FU_NBAR && (FU_CW * FU_R * 2 * 8) % 16 == 0, "fused smem layout");

struct FusedArgs {
  CostView cost;
  int64_t i0, i1;
  const double* a;        // a, a_bar (device scalars)
  const double* b[2];
  const double* rw;       // r, global row index
  int64_t* shift;         // nr: read by pass A, shift_next written by the row's finalizer
  int64_t* m_used;        // 2 x nr
  double* S;              // 2 x nr
  double* coef;           // 2 x nr x 4
  int32_t* flags;         // [count, -, (k, li)...]
  double* col;            // 2 x n (written: this launch covers every column)
  double* part;           // FU_NSLOT x FU_P x 2 x Q
  unsigned* cnt;          // npan arrival counters (zeroed before the launch)
  int32_t* err;           // set on a wait timeout (never expected)
  int64_t W, Wq;          // column tile / segment widths (even)
  int Q, units;
};

// named barrier over the consumer warps only (the producer warp never joins)
__device__ __forceinline__ void fu_sync() { asm volatile("bar.sync 2, %0;" ::"n"(FU_THREADS) : "memory"); }

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__global__ void __launch_bounds__(FU_ALL, 1) fused_sweep_kernel(const FusedArgs F) {
  extern __shared__ __align__(128) char smem[];
  char* ring = smem + TAB_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + FU_NS * FU_SLOT);
  uint64_t* empty = full + FU_NS;
  uint64_t* adone = empty + FU_NS;       // pass-A partials of this CTA written (8 arrivals)
  uint64_t* ready = adone + 1;           // [2] row constants of a panel ready (coordinator)
  uint64_t* cfree = ready + 2;           // [2] consumers done with a constants buffer (FU_CW)
  double* red = reinterpret_cast<double*>(full + FU_NBAR);          // [FU_CW][FU_R * 2]
  char* cbuf = reinterpret_cast<char*>(red + FU_CW * FU_R * 2);    // 2 x FU_CBUF
  load_table(reinterpret_cast<double*>(smem));
  if (threadIdx.x == 0) {
    for (int s = 0; s < FU_NS; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, FU_CW); }
    mbar_init(adone, FU_R * 2);
    for (int b = 0; b < 2; ++b) { mbar_init(ready + b, 1); mbar_init(cfree + b, FU_CW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto s_coef = [&](int b) { return reinterpret_cast<double*>(cbuf + b * FU_CBUF); };
  auto s_m = [&](int b) { return reinterpret_cast<uint32_t*>(cbuf + b * FU_CBUF + FU_P * 2 * 4 * 8); };
  auto s_ok = [&](int b) { return reinterpret_cast<int*>(cbuf + b * FU_CBUF + FU_P * 2 * 4 * 8 + FU_P * 2 * 4); };

  const CostView& cv = F.cost;
  const int64_t n = cv.n, nr = F.i1 - F.i0;
  const int64_t npan = (nr + FU_P - 1) / FU_P;
  const int c = blockIdx.x;
  const bool hasA = c < F.units;
  const int rb = hasA ? c / F.Q : 0, q = hasA ? c % F.Q : 0;
  const int64_t jA0 = (int64_t)q * F.Wq, jA1 = jA0 + F.Wq < n ? jA0 + F.Wq : n;
  const int nchA = jA0 < jA1 ? (int)((jA1 - jA0 + FU_CHA - 1) / FU_CHA) : 0;
  const int64_t jB0 = (int64_t)c * F.W, jB1 = jB0 + F.W < n ? jB0 + F.W : n;
  const uint32_t wB = jB0 < jB1 ? (uint32_t)((jB1 - jB0) * 8) : 0u;

  const int Q = F.Q;
  if (threadIdx.x >= FU_COORD) {  // ---------------- coordinator warp ----------------
    const int lane = threadIdx.x & 31;
    for (int64_t s = 0; s < npan + FU_LAG - 1; ++s) {
      if (s < npan && hasA) {  // publish this CTA's pass-A partials of panel s
        mbar_wait(adone, (uint32_t)(s & 1));
        if (lane == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(F.cnt + s) : "memory");
      }
      const int64_t pb = s + 1 - FU_LAG;  // prepare the constants of panel pb, streamed at step pb + LAG
      if (pb < 0 || pb >= npan) continue;
      const int b = (int)(pb & 1);
      if (pb >= 2) mbar_wait(cfree + b, (uint32_t)(((pb - 2) >> 1) & 1));
      if (lane == 0) {
        const unsigned* cp = F.cnt + pb;
        if (ld_acquire_u32(cp) < (unsigned)F.units) {
          uint64_t t0;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          while (ld_acquire_u32(cp) < (unsigned)F.units) {
            uint64_t t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            if (t1 - t0 > 4000000000ull) {  // 4 s: a co-residency failure; never expected
              atomicExch(F.err, 1);
              break;
            }
          }
        }
      }
      __syncwarp();
      const int64_t p0 = F.i0 + pb * FU_P;
      const int rows = (int)(F.i1 - p0 < FU_P ? F.i1 - p0 : FU_P);
      const int rr = lane >> 1, k = lane & 1;
      bool good = false;
      if (rr < rows) {
        const double* part = F.part + (pb % FU_NSLOT) * (FU_P * 2 * Q) + (rr * 2 + k) * Q;
        double S = __ldcg(part);
        for (int qx = 1; qx < Q; ++qx) S += __ldcg(part + qx);
        const int64_t li = p0 + rr - F.i0;
        const int64_t m = __ldcg(F.m_used + k * nr + li);
        const bool ok = sum_ok(S);
        const double g = ok ? __ldg(F.rw + p0 + rr) / S : 0.0;
        double* cf = s_coef(b) + (rr * 2 + k) * 4;
        cf[0] = g * EC0; cf[1] = g * EC1; cf[2] = g * EC2; cf[3] = g * EC3;
        s_m(b)[rr * 2 + k] = (uint32_t)m;
        s_ok(b)[rr * 2 + k] = ok ? 1 : 0;
        good = ok;
        if (c == rr % gridDim.x) {  // this CTA finalizes row rr (dxg outputs, fixup list)
          F.S[k * nr + li] = S;
          if (ok) {
            double* co = F.coef + (k * nr + li) * 4;
            co[0] = cf[0]; co[1] = cf[1]; co[2] = cf[2]; co[3] = cf[3];
            if (k == 1) F.shift[li] = m + llrint(log(S) * (1.0 / LSTEP));
          } else {
            const int slot = atomicAdd(F.flags, 1);
            F.flags[2 + 2 * slot] = k;
            F.flags[3 + 2 * slot] = (int)li;
          }
        }
      }
      // whole panel regular (16 rows, every sum in range): branch-free unrolled stages
      const unsigned all = __all_sync(0xffffffffu, good || rr >= rows) && rows == FU_P;
      if (lane == 0) {
        s_ok(b)[FU_P * 2] = all ? 1 : 0;
        s_ok(b)[FU_P * 2 + 1] = rows;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(ready + b);
    }
    return;
  }
  if (threadIdx.x >= FU_PROD) {  // ---------------- producer warp ----------------
    if (threadIdx.x == FU_PROD) {
      const uint64_t pol = l2_evict_first_policy();
      uint32_t qq = 0;
      auto acquire = [&](uint32_t bytes) -> char* {
        const int s = qq % FU_NS;
        mbar_wait(empty + s, ((qq / FU_NS) & 1) ^ 1);
        mbar_arrive_tx(full + s, bytes);
        ++qq;
        return ring + s * FU_SLOT;
      };
      for (int64_t s = 0; s < npan + FU_LAG; ++s) {
        if (s < npan && hasA) {
          const int64_t ib = F.i0 + s * FU_P + rb * FU_R;
          if (ib < F.i1) {
            for (int ch = 0; ch < nchA; ++ch) {
              const int64_t j0 = jA0 + (int64_t)ch * FU_CHA;
              const uint32_t w = (uint32_t)((jA1 - j0 < FU_CHA ? jA1 - j0 : FU_CHA) * 8);
              char* dst = acquire((FU_R + 2) * w);
              uint64_t* bar = full + ((qq - 1) % FU_NS);
#pragma unroll
              for (int r = 0; r < FU_R; ++r) {
                const int64_t i = ib + r < F.i1 ? ib + r : F.i1 - 1;
                bulk_g2s(dst + r * FU_CHA * 8, cv.mat + (i - cv.row_base) * cv.ld + j0, w, bar);
              }
              bulk_g2s(dst + FU_R * FU_CHA * 8, F.b[0] + j0, w, bar);
              bulk_g2s(dst + (FU_R + 1) * FU_CHA * 8, F.b[1] + j0, w, bar);
            }
          }
        }
        if (s >= FU_LAG && wB) {
          const int64_t p0 = F.i0 + (s - FU_LAG) * FU_P;
          const int rows = (int)(F.i1 - p0 < FU_P ? F.i1 - p0 : FU_P);
          for (int r0 = 0; r0 < rows; r0 += FU_RB) {
            const int nq = rows - r0 < FU_RB ? rows - r0 : FU_RB;
            char* dst = acquire(nq * wB);
            uint64_t* bar = full + ((qq - 1) % FU_NS);
            for (int r = 0; r < nq; ++r)
              bulk_g2s_hint(dst + r * wB, cv.mat + (p0 + r0 + r - cv.row_base) * cv.ld + jB0, wB, bar, pol);
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const uint32_t tb = lane_tab_addr(smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double na[2];
  na[0] = -F.a[0]; na[1] = -F.a[1];
  uint32_t qq = 0;  // ring position (same sequence as the producer)
  auto wait_full = [&]() -> const char* {
    const int s = qq % FU_NS;
    mbar_wait(full + s, (qq / FU_NS) & 1);
    return ring + s * FU_SLOT;
  };
  auto wait_at = [&](uint32_t q2) -> const char* {
    const int s = q2 % FU_NS;
    mbar_wait(full + s, (q2 / FU_NS) & 1);
    return ring + s * FU_SLOT;
  };
  auto release_slot = [&]() {
    release(empty + (qq % FU_NS));
    ++qq;
  };
  // pass-B column pair of this thread (n and W even: pairs are all-valid or all-invalid)
  const int64_t jb = jB0 + 2 * threadIdx.x;
  const bool hasB = jb < jB1;
  double nb[2][2], acc[2][2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    nb[k][0] = hasB ? -__ldg(F.b[k] + jb) : 0.0;
    nb[k][1] = hasB ? -__ldg(F.b[k] + jb + 1) : 0.0;
    acc[k][0] = 0.0; acc[k][1] = 0.0;
  }

  for (int64_t s = 0; s < npan + FU_LAG; ++s) {
    // ---- pass A: row partial sums of this CTA's unit of panel s ----
    if (s < npan && hasA) {
      const int64_t ib = F.i0 + s * FU_P + rb * FU_R;
      double* part = F.part + (s % FU_NSLOT) * (FU_P * 2 * Q);
      if (ib < F.i1) {
        uint32_t mlo[FU_R];
#pragma unroll
        for (int r = 0; r < FU_R; ++r) {
          const int64_t i = ib + r < F.i1 ? ib + r : F.i1 - 1;
          mlo[r] = (uint32_t)F.shift[i - F.i0];
        }
        double sa[FU_R][2];
#pragma unroll
        for (int r = 0; r < FU_R; ++r) { sa[r][0] = 0.0; sa[r][1] = 0.0; }
        for (int ch = 0; ch < nchA; ++ch) {
          const char* st = wait_full();
          const int64_t j = jA0 + (int64_t)ch * FU_CHA + 2 * threadIdx.x;
          if (j < jA1) {
            const char* p = st + 16 * threadIdx.x;
            const double2 bv0 = *reinterpret_cast<const double2*>(p + FU_R * FU_CHA * 8);
            const double2 bv1 = *reinterpret_cast<const double2*>(p + (FU_R + 1) * FU_CHA * 8);
#pragma unroll
            for (int r = 0; r < FU_R; ++r) {
              const double2 cc = *reinterpret_cast<const double2*>(p + r * FU_CHA * 8);
              texp_acc(tb, fma(na[0], cc.x, -bv0.x), mlo[r], sa[r][0]);
              texp_acc(tb, fma(na[0], cc.y, -bv0.y), mlo[r], sa[r][0]);
              texp_acc(tb, fma(na[1], cc.x, -bv1.x), mlo[r], sa[r][1]);
              texp_acc(tb, fma(na[1], cc.y, -bv1.y), mlo[r], sa[r][1]);
            }
          }
          release_slot();
        }
        // transpose-reduce of the 8 row sums over the warp (9 SHFL + 9 DADD instead of 40):
        // after the halving levels 16/8/4, lane L holds value (L >> 2) & 7 summed over
        // the 8 lanes that differ in bits 4..2; levels 2/1 finish the sum (fixed order)
        {
          const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
          double w[4], u[2];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double keep = b4 ? sa[(i + 4) >> 1][(i + 4) & 1] : sa[i >> 1][i & 1];
            const double send = b4 ? sa[i >> 1][i & 1] : sa[(i + 4) >> 1][(i + 4) & 1];
            w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const double keep = b3 ? w[i + 2] : w[i];
            const double send = b3 ? w[i] : w[i + 2];
            u[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
          }
          double x = (b2 ? u[1] : u[0]) + __shfl_xor_sync(0xffffffffu, b2 ? u[0] : u[1], 4);
          x += __shfl_xor_sync(0xffffffffu, x, 2);
          x += __shfl_xor_sync(0xffffffffu, x, 1);
          if ((lane & 3) == 0) red[warp * (FU_R * 2) + (lane >> 2)] = x;
        }
        fu_sync();
        if (threadIdx.x < FU_R * 2) {
          const int r = threadIdx.x >> 1, k = threadIdx.x & 1;
          double t = red[threadIdx.x];
          for (int w = 1; w < FU_CW; ++w) t += red[w * (FU_R * 2) + threadIdx.x];
          part[((rb * FU_R + r) * 2 + k) * Q + q] = t;
          const int64_t i = ib + r;
          if (q == 0 && i < F.i1) F.m_used[k * nr + (i - F.i0)] = F.shift[i - F.i0];
        }
      }
      // the 8 writers signal the coordinator, which publishes the unit at gpu scope
      if (threadIdx.x < FU_R * 2) mbar_arrive(adone);
    }
    // ---- pass B: column sums of this CTA's tile over panel s-LAG ----
    if (s >= FU_LAG) {
      const int64_t pb = s - FU_LAG;
      const int b = (int)(pb & 1);
      mbar_wait(ready + b, (uint32_t)((pb >> 1) & 1));
      const double* coef = s_coef(b);
      const uint32_t* sm = s_m(b);
      const int* so = s_ok(b);
      const bool fast = so[FU_P * 2] != 0;
      const int rows = so[FU_P * 2 + 1];
      if (wB && fast) {
        // regular panel: two stages (8 rows) per round for more independent exps per thread
        for (int r0 = 0; r0 < FU_P; r0 += 2 * FU_RB) {
          const char* st0 = wait_at(qq);
          const char* st1 = wait_at(qq + 1);
          if (hasB) {
            double2 cc[2 * FU_RB];
#pragma unroll
            for (int r = 0; r < 2 * FU_RB; ++r)
              cc[r] = *reinterpret_cast<const double2*>((r < FU_RB ? st0 : st1) + 16 * threadIdx.x + (r % FU_RB) * wB);
#pragma unroll
            for (int r = 0; r < 2 * FU_RB; ++r)
#pragma unroll
              for (int k = 0; k < 2; ++k) {
                const int rr = r0 + r;
                const double2 g01 = *reinterpret_cast<const double2*>(coef + (rr * 2 + k) * 4);
                const double2 g23 = *reinterpret_cast<const double2*>(coef + (rr * 2 + k) * 4 + 2);
                const uint32_t ml = sm[rr * 2 + k];
                texp_gacc(tb, fma(na[k], cc[r].x, nb[k][0]), ml, g01.x, g01.y, g23.x, g23.y, acc[k][0]);
                texp_gacc(tb, fma(na[k], cc[r].y, nb[k][1]), ml, g01.x, g01.y, g23.x, g23.y, acc[k][1]);
              }
          }
          release_slot();
          release_slot();
        }
      } else if (wB) {
        for (int r0 = 0; r0 < rows; r0 += FU_RB) {
          const char* st = wait_full();
          const int nq = rows - r0 < FU_RB ? rows - r0 : FU_RB;
          if (hasB) {
            const char* p = st + 16 * threadIdx.x;
            for (int r = 0; r < nq; ++r) {
              const double2 cc = *reinterpret_cast<const double2*>(p + r * wB);
              const int rr = r0 + r;
#pragma unroll
              for (int k = 0; k < 2; ++k) {
                if (so[rr * 2 + k]) {
                  const double2 g01 = *reinterpret_cast<const double2*>(coef + (rr * 2 + k) * 4);
                  const double2 g23 = *reinterpret_cast<const double2*>(coef + (rr * 2 + k) * 4 + 2);
                  const uint32_t ml = sm[rr * 2 + k];
                  texp_gacc(tb, fma(na[k], cc.x, nb[k][0]), ml, g01.x, g01.y, g23.x, g23.y, acc[k][0]);
                  texp_gacc(tb, fma(na[k], cc.y, nb[k][1]), ml, g01.x, g01.y, g23.x, g23.y, acc[k][1]);
                }
              }
            }
          }
          release_slot();
        }
      }
      release(cfree + b);  // this warp is done with the panel's constants
    }
  }
  if (hasB) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      F.col[k * n + jb] = acc[k][0];
      F.col[k * n + jb + 1] = acc[k][1];
    }
  }
}

// Rows flagged by the fused sweep: exact max shift, row sum, the row's outputs (as
// fixup_kernel) and its column contributions, which pass B skipped.  One CTA, flagged
// (k, row) entries in ascending order (sorted here), so the result is deterministic.
__global__ void __launch_bounds__(1024) fused_fix_kernel(const FusedArgs F) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double red[32];
  __shared__ double bcast;
  const int cnt = *F.flags;
  if (cnt == 0) return;
  load_table(reinterpret_cast<double*>(smem));
  if (threadIdx.x == 0) {  // insertion sort of the (k, li) list (rare, short)
    for (int e = 1; e < cnt; ++e) {
      const int k = F.flags[2 + 2 * e], l = F.flags[3 + 2 * e];
      int f = e - 1;
      while (f >= 0 && (F.flags[2 + 2 * f] > k || (F.flags[2 + 2 * f] == k && F.flags[3 + 2 * f] > l))) {
        F.flags[4 + 2 * f] = F.flags[2 + 2 * f];
        F.flags[5 + 2 * f] = F.flags[3 + 2 * f];
        --f;
      }
      F.flags[4 + 2 * f] = k;
      F.flags[5 + 2 * f] = l;
    }
  }
  __syncthreads();
  const uint32_t tb = lane_tab_addr(smem);
  const CostView& cv = F.cost;
  const int64_t n = cv.n, nr = F.i1 - F.i0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = 0; e < cnt; ++e) {
    const int k = F.flags[2 + 2 * e];
    const int64_t li = F.flags[3 + 2 * e];
    const double* row = cv.mat + (F.i0 + li - cv.row_base) * cv.ld;
    const double na = -F.a[k];
    double mx = -INFINITY;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) mx = fmax(mx, fma(na, row[j], -F.b[k][j]));
    mx = warp_max(mx);
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red[0];
      for (int w = 1; w < nw; ++w) t = fmax(t, red[w]);
      bcast = t;
    }
    __syncthreads();
    const int64_t m = llrint(bcast * (1.0 / LSTEP));
    const uint32_t mlo = (uint32_t)m;
    double s = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) texp_acc(tb, fma(na, row[j], -F.b[k][j]), mlo, s);
    s = warp_sum(s);
    __syncthreads();
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red[0];
      for (int w = 1; w < nw; ++w) t += red[w];
      bcast = t;
      F.S[k * nr + li] = t;
      F.m_used[k * nr + li] = m;
      const double g = __ldg(F.rw + F.i0 + li) / t;
      double* co = F.coef + (k * nr + li) * 4;
      co[0] = g * EC0; co[1] = g * EC1; co[2] = g * EC2; co[3] = g * EC3;
      if (k == 1) F.shift[li] = m + llrint(log(t) * (1.0 / LSTEP));
    }
    __syncthreads();
    const double g = __ldg(F.rw + F.i0 + li) / bcast;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x)
      texp_gacc(tb, fma(na, row[j], -F.b[k][j]), mlo, g * EC0, g * EC1, g * EC2, g * EC3, F.col[k * n + j]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *F.flags = 0;
}

// LEANOT_FUSED=1 makes the fused sweep the default for plain iterations (experiments);
// otherwise it runs only when asked for with LEANOT_SWEEP_FUSED
static bool fused_default() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LEANOT_FUSED");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// Launch the fused sweep for a DXG plan if it applies (stored cost on the TMA path, all
// weight sets of a plain iteration, n in [16384, 148 x 1056]); returns LEANOT_OK when it
// ran, LEANOT_EINVAL when the caller should use the two-pass sweep.
static int try_fused_sweep(const leanot_dxg_plan_t& P, cudaStream_t st) {
  const CostView cv = make_view(P.cost);
  if (!tma_ok(cv) || P.n < 16384) return LEANOT_EINVAL;
  const int G = num_sms();
  constexpr int UPP = FU_P / FU_R;  // units per panel row block
  const int Q = G / UPP;
  if (Q < 1) return LEANOT_EINVAL;
  const int64_t W = (((P.n + G - 1) / G) + 1) & ~int64_t(1);
  const int64_t Wq = (((P.n + Q - 1) / Q) + 1) & ~int64_t(1);
  if (W > FU_WMAX || W / 2 > FU_THREADS) return LEANOT_EINVAL;
  const int64_t nr = P.row1 - P.row0, npan = (nr + FU_P - 1) / FU_P;
  // scratch carved from the (unused) column slab: partial sums, counters, error flag
  const int64_t part_d = (int64_t)FU_NSLOT * FU_P * 2 * Q;
  const int64_t cnt_d = (npan + 2 + 1) / 2 + 1;
  if (part_d + cnt_d > (int64_t)P.splits * 2 * P.n) return LEANOT_EINVAL;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(fused_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FU_SMEM) != cudaSuccess)
      return LEANOT_EINVAL;
    if (cudaFuncSetAttribute(fused_fix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TAB_BYTES) != cudaSuccess)
      return LEANOT_EINVAL;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fused_sweep_kernel, FU_ALL, FU_SMEM) != cudaSuccess ||
        occ < 1)
      return LEANOT_EINVAL;
    attr = true;
  }
  FusedArgs F;
  memset(&F, 0, sizeof(F));
  F.cost = cv;
  F.i0 = P.row0; F.i1 = P.row1;
  F.a = P.scal;
  F.b[0] = P.b; F.b[1] = P.b_bar;
  F.rw = P.r;
  F.shift = P.shift; F.m_used = P.m; F.S = P.S; F.coef = P.coef;
  F.flags = P.flags; F.col = P.col;
  F.part = P.slab;
  F.cnt = reinterpret_cast<unsigned*>(P.slab + part_d);
  F.err = reinterpret_cast<int32_t*>(F.cnt + npan);
  F.W = W; F.Wq = Wq; F.Q = Q; F.units = Q * UPP;
  cudaMemsetAsync(F.cnt, 0, (npan + 1) * sizeof(unsigned), st);
  cudaLaunchConfig_t lc;
  memset(&lc, 0, sizeof(lc));
  lc.gridDim = dim3(G);
  lc.blockDim = dim3(FU_ALL);
  lc.dynamicSmemBytes = FU_SMEM;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&lc, fused_sweep_kernel, F);
  if (e != cudaSuccess) {
    set_error("fused sweep launch: %s", cudaGetErrorString(e));
    return LEANOT_ECUDA;
  }
  fused_fix_kernel<<<1, 1024, TAB_BYTES, st>>>(F);
  return LEANOT_OK;
}

}  // namespace leanot
