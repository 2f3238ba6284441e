// Single-read, single-exp DXG sweep for the stored cost (BASELINE config 3 path).
//
// One DXG iteration needs both column marginals of the current state (dxg.py:272, :276):
//   col_kj = sum_i r_i exp(x_kij - L_ki),  x_kij = -(a_k C_ij + b_kj),  k in {now, bar}
// (column_marginal, dxg.py:193-208).  The row normalizer L_ki must be complete before row
// i's column contributions can be accumulated, so the two-pass sweep reads C twice and
// evaluates every exponential twice (4 exps per element per iteration).  This kernel
// reads each element of C once and evaluates each exponential once (2 per element):
//
//   * G = #SMs persistent CTAs (cooperative launch: all co-resident).  CTA c owns the
//     column tile [c W, (c+1) W) (W ~ n/G, <= 2 x 352) for ALL rows of the sweep; each
//     of its 352 consumer threads owns 2 adjacent columns, so the column sums live in
//     registers for the whole launch (no slabs, no second-stage reduce).
//   * Rows stream in panels of P rows: the panel's C tile rows (W doubles each) and row
//     shifts arrive in a shared-memory ring by cp.async.bulk, issued by consumer thread 0
//     right after the per-panel consumer barrier has retired the slot (no producer warp:
//     12 warps keep the 168-register budget that holds D panels of exps).  The consumers
//     evaluate e_kij = exp(x_kij - m_i LSTEP) for both weight sets, KEEP the exps in
//     registers, and reduce their row partial sums (warp shuffles, then warps in fixed
//     order) into one partial per (row, set) per CTA.
//   * Exchange: each CTA publishes its 2P partials of panel p into a global slot; a
//     collector warp in every CTA reads all G partials of the panel and sums them in the
//     same fixed order, so every CTA obtains bitwise the same S_ki = sum_j e_kij.  Every
//     8-byte partial carries its slot generation in the sign bit (partials are >= 0), so
//     a value is its own ready flag: no fences, one L2 round trip.
//   * D panels of exps stay in registers while the exchange is in flight; after panel p
//     is computed, panel p-D+1 is folded into the column sums with g_i = r_i / S_ki
//     (acc_kj += g_ki e_kij: one FMA per element and set).
//   FP64 work per element and weight set: 9.5 instructions (affine, 7 of the table exp,
//   half a row-sum add, the column FMA) instead of 2 x 8 in the two-pass form.
//
// Rows whose sum leaves [2^-900, 2^900] are skipped (g = 0) and recomputed exactly
// afterwards in ascending order (fused_fix_kernel), as in the other sweeps.  Outputs:
// col (2 x n, complete for the local rows), S and m_used (2 x nr), the next iteration's
// shifts (from the midpoint set, as finalize_row), the fixup list.  Deterministic: fixed
// reduction orders everywhere, no floating-point atomics.  Every spin loop has a 4 s
// timeout that sets an error flag and drains the launch (never expected).
// Included by leanot_lib.cu after leanot_fused.cu (mbarrier / bulk-copy helpers).

namespace leanot {

constexpr int SR_CW = 11;                    // consumer warps
constexpr int SR_THREADS = SR_CW * 32;       // 352 consumer threads, 2 columns each
constexpr int SR_WMAX = 2 * SR_THREADS;      // 704: widest column tile
constexpr int SR_COLL = SR_THREADS;          // collector warp
constexpr int SR_ALL = SR_THREADS + 32;      // 12 warps: 168 registers per thread
constexpr int SR_NS = 6;                     // C ring slots (one panel each; 4 left ~6 % C-data waits at full HBM load)
constexpr int SR_NSLOT = 16;                 // partial-sum slots in flight (>= 2 D)
constexpr int SR_CPC = 40;                   // max CTAs per collector chunk (G <= 4 x 40)
constexpr int SR_NR = 4;                     // per-warp row-sum buffers in flight (>= D + 1)
constexpr uint64_t SR_TIMEOUT_NS = 4000000000ull;

template <int P>
struct SrLayout {
  static constexpr int NV = 2 * P;                      // (row, set) partials per panel
  static constexpr int ROWB = SR_WMAX * 8;              // bytes per staged row
  static constexpr int HDR = 64;                        // shift values of the panel (P <= 8)
  static constexpr int SLOT = HDR + P * ROWB;
  static constexpr int RING = TAB_BYTES;                // ring after the exp table
  static constexpr int RED = RING + SR_NS * SLOT;       // [SR_NR][CW][NV] doubles
  static constexpr int WB = RED + SR_NR * SR_CW * NV * 8;  // [D][NV] doubles + [D][NV + 1] ints (<= 8 D)
  static constexpr int BAR = WB + 8 * (NV * 8 + (NV + 1) * 4 + 8);  // mbarriers (up to 8 D slots)
  static constexpr int SMEM = BAR + 8 * (2 * SR_NS + 16) + 16;
  static_assert(P <= 4 && (32 % NV) == 0, "SR panel shape (collector buffers hold 2P <= 8 values per CTA)");
};

struct SrArgs {
  CostView cost;
  int64_t i0, i1;
  const double* a;        // a, a_bar (device scalars)
  const double* b[2];
  const double* rw;       // r, global row index
  int64_t* shift;         // nr: read for the sweep, overwritten with the next sweep's shifts
  int64_t* m_used;        // 2 x nr
  double* S;              // 2 x nr
  double* coef;           // 2 x nr x 4 (written only by the fixup)
  int32_t* flags;         // [count, -, (k, li)...]
  double* col;            // 2 x n
  unsigned long long* part;  // SR_NSLOT x G x NV tagged partials (0xff-filled before the launch)
  int32_t* err;
  int64_t W;              // column tile width (even)
  unsigned long long* trace;  // debug (null in production): per-panel timestamps of CTAs 0 and G-1
};

__device__ __forceinline__ uint64_t sr_now() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// mbarrier wait that gives up after SR_TIMEOUT_NS (sets *abort; later waits return at once).
// try_wait carries a suspend-time hint, so a waiting warp sleeps in hardware instead of
// spinning (it would otherwise take issue slots from the warps it waits for).
__device__ __forceinline__ bool sr_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void sr_wait(uint64_t* bar, uint32_t parity, volatile int* abort) {
  if (sr_try(bar, parity)) return;
  uint64_t t0 = 0;
  for (uint32_t spin = 1;; ++spin) {
    if (sr_try(bar, parity)) return;
    if ((spin & 255) == 0) {   // the clock and the abort flag are consulted every 256 polls
      if (*abort) return;
      const uint64_t t = sr_now();
      if (t0 == 0) t0 = t;
      else if (t - t0 > SR_TIMEOUT_NS) { *abort = 1; return; }
    }
  }
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// sum over the warp of NV per-lane values; lane (v * 32 / NV) ends up with the sum of value v
// (transpose-reduce: log2(NV) halving exchanges, then plain butterflies; fixed order)
template <int NV>
__device__ __forceinline__ double warp_transpose_sum(double (&x)[NV], int lane) {
  if constexpr (NV == 8) {
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
    double w[4], u[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double keep = b4 ? x[i + 4] : x[i];
      const double send = b4 ? x[i] : x[i + 4];
      w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const double keep = b3 ? w[i + 2] : w[i];
      const double send = b3 ? w[i] : w[i + 2];
      u[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    double y = (b2 ? u[1] : u[0]) + __shfl_xor_sync(0xffffffffu, b2 ? u[0] : u[1], 4);
    y += __shfl_xor_sync(0xffffffffu, y, 2);
    y += __shfl_xor_sync(0xffffffffu, y, 1);
    return y;  // lane L holds value (L >> 2): value v at lane 4 v
  } else if constexpr (NV == 4) {
    const bool b4 = lane & 16, b3 = lane & 8;
    double w[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const double keep = b4 ? x[i + 2] : x[i];
      const double send = b4 ? x[i] : x[i + 2];
      w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    double y = (b3 ? w[1] : w[0]) + __shfl_xor_sync(0xffffffffu, b3 ? w[0] : w[1], 8);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
    return y;  // lane L holds value (L >> 3): value v at lane 8 v
  } else {
    static_assert(NV == 2, "NV");
    const bool b4 = lane & 16;
    double y = (b4 ? x[1] : x[0]) + __shfl_xor_sync(0xffffffffu, b4 ? x[0] : x[1], 16);
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
    return y;  // value v at lane 16 v
  }
}

template <int P, int D, bool TRACE>
__global__ void __launch_bounds__(SR_ALL, 1) sr_sweep_kernel(const SrArgs F) {
  using L = SrLayout<P>;
  constexpr int NV = L::NV;
  extern __shared__ __align__(128) char smem[];
  char* ring = smem + L::RING;
  double* red = reinterpret_cast<double*>(smem + L::RED);
  double* wbuf = reinterpret_cast<double*>(smem + L::WB);          // [D][NV]
  int* okbuf = reinterpret_cast<int*>(wbuf + D * NV);               // [D][NV + 1] (last: all ok)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* wready = full + SR_NS;
  uint64_t* wfree = wready + D;
  volatile int* s_abort = reinterpret_cast<volatile int*>(wfree + D);
  int* s_cnt = reinterpret_cast<int*>(wfree + D + 1);               // [SR_NR] warps done with a panel
  static_assert(SR_NS + 2 * D + 1 + SR_NR / 2 <= 2 * SR_NS + 16 && SR_NR >= D + 1, "SR barriers");
  load_table(reinterpret_cast<double*>(smem));
  if (threadIdx.x == 0) {
    for (int s = 0; s < SR_NS; ++s) mbar_init(full + s, 1);
    for (int s = 0; s < D; ++s) { mbar_init(wready + s, 1); mbar_init(wfree + s, SR_CW); }
    *s_abort = 0;
    for (int i = 0; i < SR_NR; ++i) s_cnt[i] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const CostView& cv = F.cost;
  const int64_t n = cv.n, nr = F.i1 - F.i0;
  const int64_t npan = (nr + P - 1) / P;
  const int G = gridDim.x, c = blockIdx.x;
  const int64_t j0 = (int64_t)c * F.W, j1 = j0 + F.W < n ? j0 + F.W : n;
  const uint32_t wbytes = j0 < j1 ? (uint32_t)((j1 - j0) * 8) : 0u;
  const int lane = threadIdx.x & 31;
  // debug trace (clock64 of this SM), trace[q*8 + e]: 0 own partial published, 1 collector
  // iteration start, 2 prefetched buffer ready, 3 re-polls done, 4 g posted, 5 consumer starts
  // waiting for g, 6 consumer got g, 7 number of re-poll rounds
  unsigned long long* trace =
      TRACE && F.trace && (c == 0 || c == G - 1) ? F.trace + (c == 0 ? 0 : 8 * 4096) : nullptr;
  if (!TRACE || npan > 4096) trace = nullptr;

  if (threadIdx.x >= SR_COLL) {  // ------------------------- collector warp -------------------------
    // Layout of a panel's partials: [CTA c][v = 2 r + k].  Lane l loads 16-byte pairs at
    // doubles 2 l + 64 jj: values v0 = 2 (l % 4), v0 + 1 of CTA 8 jj + l / 4, so lanes l, l ^ 4,
    // l ^ 8, l ^ 16 hold the same two values of different CTAs and three butterfly levels
    // finish the sums.  The order (jj ascending per lane, then the butterfly) is fixed, so
    // every CTA computes bitwise the same S.
    // Generation tags: a value of parity `par` carries sign bit `par`; the raw doubles are
    // summed as they are (for par = 1 every term is negated, so S = -sum exactly) and a load
    // is stale if any value's sign bit differs (OR of high words ^ parity bit).
    // The loads are direct relaxed loads, all in flight at once (LSU path: they do not queue
    // behind the C-tile bulk copies in the SM's TMA unit), and software-pipelined: panel
    // q + 1's loads are issued before panel q's S are finalized, so the L2 round trip
    // overlaps the finalization.
    static_assert(NV == 8, "collector layout assumes P = 4");
    constexpr int NJ = (4 * SR_CPC * 8) / 64;              // 16-byte loads per lane covering G <= 160
    const int cl = lane >> 2;                              // CTA offset within a group of 8
    const int njj = (G + 7) / 8;
    bool dead = false;
    double2 y[NJ];
    auto issue = [&](int64_t q) {
      const double2* gp = reinterpret_cast<const double2*>(F.part + (q % SR_NSLOT) * G * NV) + lane;
#pragma unroll
      for (int jj = 0; jj < NJ; ++jj)
        if (jj < njj && 8 * jj + cl < G) {
          unsigned long long u0, u1;
          asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(u0), "=l"(u1) : "l"(gp + 32 * jj));
          y[jj] = make_double2(__longlong_as_double((long long)u0), __longlong_as_double((long long)u1));
        }
    };
    if (npan > 0) issue(0);
    // lanes 0..3 finalize row r = lane of each panel: r_i prefetched one panel ahead
    double rw_next = (lane < P && lane < nr) ? __ldg(F.rw + F.i0 + lane) : 0.0;
    for (int64_t q = 0; q < npan; ++q) {
      const unsigned long long parbits = (unsigned long long)((q / SR_NSLOT) & 1) << 63;
      const double rw_q = rw_next;
      if (q + 1 < npan && lane < P) {
        const int64_t li1 = (q + 1) * P + lane;
        rw_next = li1 < nr ? __ldg(F.rw + F.i0 + li1) : 0.0;
      }
      if (TRACE && trace && lane == 0) trace[q * 8 + 1] = clock64();
      double a0, a1, c0, c1;   // (v0, v1) x (even jj, odd jj)
      const uint64_t t0 = sr_now();
      int rounds = 0;
      while (true) {
        a0 = a1 = c0 = c1 = 0.0;
        // sign bits only: one 3-input LOP per value on the high words
        const unsigned p32 = (unsigned)(parbits >> 32);
        unsigned bad = 0;
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj)
          if (jj < njj && 8 * jj + cl < G) {
            bad |= ((unsigned)__double2hiint(y[jj].x) ^ p32);
            bad |= ((unsigned)__double2hiint(y[jj].y) ^ p32);
            if (jj & 1) { c0 += y[jj].x; c1 += y[jj].y; } else { a0 += y[jj].x; a1 += y[jj].y; }
          }
        if (!__any_sync(0xffffffffu, bad >> 31) || dead) break;
        // some CTA had not published panel q when the loads ran: poll again
        ++rounds;
        const uint64_t el = sr_now() - t0;
        if (__any_sync(0xffffffffu, el > SR_TIMEOUT_NS || (el > 1000000ull && *(volatile int32_t*)F.err != 0))) {
          dead = true;   // co-residency / protocol failure (never expected): report and drain
          if (lane == 0) atomicExch(F.err, 1);
          break;
        }
        issue(q);
      }
      if (q + 1 < npan) issue(q + 1);   // next panel's round trip overlaps this finalization
      if (TRACE && trace && lane == 0) { trace[q * 8 + 2] = clock64(); trace[q * 8 + 7] = rounds; }
      double s0 = a0 + c0, s1 = a1 + c1;
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      }
      if (parbits) { s0 = -s0; s1 = -s1; }
      if (TRACE && trace && lane == 0) trace[q * 8 + 3] = clock64();
      // lanes 0..3: row r = lane, S0 = S of the current weights, S1 = S of the midpoint weights
      const int64_t li = q * P + lane;
      const bool valid = lane < P && li < nr;
      const bool ok0 = valid && sum_ok(s0) && !dead, ok1 = valid && sum_ok(s1) && !dead;
      // g = r_i / S: one correctly rounded reciprocal and a multiply (<= 1.5 ulp of the quotient)
      const double w0 = ok0 ? rw_q * __drcp_rn(s0) : 0.0, w1 = ok1 ? rw_q * __drcp_rn(s1) : 0.0;
      const int ds = (int)(q % D);
      if (q >= D) sr_wait(wfree + ds, (uint32_t)(((q / D) - 1) & 1), s_abort);
      if (lane < P) {
        wbuf[ds * NV + 2 * lane] = w0;
        wbuf[ds * NV + 2 * lane + 1] = w1;
        okbuf[ds * (NV + 1) + 2 * lane] = ok0 ? 1 : 0;
        okbuf[ds * (NV + 1) + 2 * lane + 1] = ok1 ? 1 : 0;
      }
      const bool all = __all_sync(0xffffffffu, lane >= P || (ok0 && ok1));
      if (lane == 0) okbuf[ds * (NV + 1) + NV] = all ? 1 : 0;
      __syncwarp();
      if (TRACE && trace && lane == 0) trace[q * 8 + 4] = clock64();
      if (lane == 0) mbar_arrive(wready + ds);
      if (valid && (int)(q % G) == c) {  // this CTA finalizes the panel's rows (off the consumers' path)
        const int64_t m = F.shift[li];
        F.S[li] = s0;
        F.S[nr + li] = s1;
        F.m_used[li] = m;
        F.m_used[nr + li] = m;
        if (!ok0 || !ok1) {
          const int nf = (ok0 ? 0 : 1) + (ok1 ? 0 : 1);
          int slot2 = atomicAdd(F.flags, nf);
          if (!ok0) { F.flags[2 + 2 * slot2] = 0; F.flags[3 + 2 * slot2] = (int)li; ++slot2; }
          if (!ok1) { F.flags[2 + 2 * slot2] = 1; F.flags[3 + 2 * slot2] = (int)li; }
        }
        if (ok1) F.shift[li] = m + llrint(log(s1) * (1.0 / LSTEP));
      }
      __syncwarp();
    }
    return;
  }
  // ------------------------------ consumers ------------------------------
  const uint32_t tb = lane_tab_addr(smem);
  const int warp = threadIdx.x >> 5;
  // Column group of this warp.  Warp w issues on SMSP w % 4; the collector (warp 11) shares
  // SMSP 3 with warps 3 and 7, so warp 7 takes the LAST column group, which is only partly
  // filled when W < 704 (n = 1e5: 36 of 64 columns), leaving the collector issue slots.
  const int cgrp = warp == 7 ? SR_CW - 1 : (warp == SR_CW - 1 ? 7 : warp);
  const int tcol = cgrp * 32 + lane;
  const int64_t jt = 2 * tcol;                  // local column pair
  const bool has = j0 + jt < j1;                // n and W even: pairs are whole
  double na[2], nb[2][2], acc[2][2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    na[k] = -F.a[k];
    nb[k][0] = has ? -__ldg(F.b[k] + j0 + jt) : 0.0;
    nb[k][1] = has ? -__ldg(F.b[k] + j0 + jt + 1) : 0.0;
    acc[k][0] = 0.0; acc[k][1] = 0.0;
  }
  double e[D][P][2][2];
  uint32_t s = 0, ph = 0;
  // thread 0: fill ring slot `slot` with panel p (row shifts + the C tile rows)
  auto refill = [&](int p, int slot) {
    const int64_t li0 = p * P;
    const int rows = (int)(nr - li0 < P ? nr - li0 : P);
    char* dst = ring + slot * L::SLOT;
    uint64_t* bar = full + slot;
    if (rows < P) {  // last, partial panel: plain loads (a bulk copy would read past nr)
      int64_t* hdr = reinterpret_cast<int64_t*>(dst);
#pragma unroll
      for (int r = 0; r < P; ++r) hdr[r] = F.shift[li0 + (r < rows ? r : rows - 1)];
      mbar_arrive_tx(bar, (uint32_t)P * wbytes);
    } else {
      mbar_arrive_tx(bar, (uint32_t)P * wbytes + P * 8);
      bulk_g2s(dst, F.shift + li0, P * 8, bar);
    }
    if (wbytes) {
#pragma unroll
      for (int r = 0; r < P; ++r) {
        const int64_t i = F.i0 + li0 + (r < rows ? r : rows - 1);
        bulk_g2s(dst + L::HDR + r * L::ROWB, cv.mat + (i - cv.row_base) * cv.ld + j0, wbytes, bar);
      }
    }
  };
  if (threadIdx.x == 0)
    for (int q = 0; q < SR_NS && q < npan; ++q) refill(q, q);
  // running panel bookkeeping (32-bit, no divisions in the loop): reduction buffer pr = p % NR,
  // partial-sum slot ps = p % NSLOT with generation parity pp
  int pr = 0, ps = 0;
  unsigned long long pp = 0;
  const int npan32 = (int)npan;
  auto compute = [&](int p, double (&E)[P][2][2]) {
    sr_wait(full + s, ph, s_abort);
    const char* st = ring + s * L::SLOT;
    double rs[NV];
    {
      // threads without columns (the last CTA's tail) compute on column pair 0 of the slot and
      // contribute 0 to the row sums: no divergent zero-filling of the exps (their column sums
      // are never written)
      const uint32_t* hdr = reinterpret_cast<const uint32_t*>(st);  // int64 shifts: low words at 2r
      const int tc = has ? tcol : 0;
#pragma unroll
      for (int r = 0; r < P; ++r) {
        const uint32_t ml = hdr[2 * r];
        const double2 cc = *reinterpret_cast<const double2*>(st + L::HDR + r * L::ROWB + 16 * tc);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          E[r][k][0] = texp(tb, fma(na[k], cc.x, nb[k][0]), ml);
          E[r][k][1] = texp(tb, fma(na[k], cc.y, nb[k][1]), ml);
          rs[r * 2 + k] = has ? E[r][k][0] + E[r][k][1] : 0.0;
        }
      }
    }
    const int used = (int)s;
    if (++s == SR_NS) { s = 0; ph ^= 1; }
    // Row sums of the panel: warp transpose-reduce, then the LAST warp to finish the panel
    // (smem counter) adds the CTA's warps in fixed order, publishes the CTA partials and
    // refills the ring slot every warp has now read -- no CTA-wide barrier, so warps drift
    // apart and one warp's reduction latency overlaps the others' exps.
    const double y = warp_transpose_sum<NV>(rs, lane);
    double* rb = red + pr * (SR_CW * NV);
    if ((lane & (32 / NV - 1)) == 0) rb[warp * NV + lane / (32 / NV)] = y;
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      __threadfence_block();
      last = atomicAdd(s_cnt + pr, 1) == SR_CW - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      __threadfence_block();
      if (lane == 0) {
        s_cnt[pr] = 0;   // reused NR panels later, after this CTA's partial of p + 1 is out
        if (p + SR_NS < npan32) refill(p + SR_NS, used);
      }
      if (lane < NV) {
        const volatile double* vb = rb;
        double t = vb[lane];
#pragma unroll
        for (int w = 1; w < SR_CW; ++w) t += vb[w * NV + lane];
        const unsigned long long bits = ((unsigned long long)__double_as_longlong(t) & 0x7fffffffffffffffull) | pp;
        st_relaxed_u64(F.part + (ps * G + c) * NV + lane, bits);
        if (TRACE && trace && lane == 0) trace[p * 8] = clock64();
      }
    }
    if (++pr == SR_NR) pr = 0;
    if (++ps == SR_NSLOT) { ps = 0; pp ^= 1ull << 63; }
  };
  // fold panel q (exps E, slot ds = q % D, wready parity wpar) into the column sums
  auto accumulate = [&](int q, const double (&E)[P][2][2], int ds, uint32_t wpar) {
    if (TRACE && trace && threadIdx.x == 0) trace[q * 8 + 5] = clock64();
    sr_wait(wready + ds, wpar, s_abort);
    if (TRACE && trace && threadIdx.x == 0) trace[q * 8 + 6] = clock64();
    const double* wq = wbuf + ds * NV;
    const int* oq = okbuf + ds * (NV + 1);
    if (oq[NV]) {
#pragma unroll
      for (int r = 0; r < P; ++r)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const double g = wq[r * 2 + k];
          acc[k][0] = fma(g, E[r][k][0], acc[k][0]);
          acc[k][1] = fma(g, E[r][k][1], acc[k][1]);
        }
    } else {
#pragma unroll
      for (int r = 0; r < P; ++r)
#pragma unroll
        for (int k = 0; k < 2; ++k)
          if (oq[r * 2 + k]) {
            const double g = wq[r * 2 + k];
            acc[k][0] = fma(g, E[r][k][0], acc[k][0]);
            acc[k][1] = fma(g, E[r][k][1], acc[k][1]);
          }
    }
    release(wfree + ds);
  };
  // p0 steps by D, so panel p = p0 + u keeps its exps in e[u] and panel q = p - (D - 1) is in
  // e[(u + 1) % D] with wready slot (u + 1) % D; its use index q / D is p0 / D for u = D - 1
  // and p0 / D - 1 otherwise (phase bit wph tracks p0 / D)
  uint32_t wph = 0;
  for (int p0 = 0; p0 < npan32 + D - 1; p0 += D, wph ^= 1) {
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const int p = p0 + u;
      if (p < npan32) compute(p, e[u]);
      const int q = p - (D - 1);
      if (q >= 0 && q < npan32) accumulate(q, e[(u + 1) % D], (u + 1) % D, u == D - 1 ? wph : wph ^ 1);
    }
  }
  if (has) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      F.col[k * n + j0 + jt] = acc[k][0];
      F.col[k * n + j0 + jt + 1] = acc[k][1];
    }
  }
  if (*s_abort && threadIdx.x == 0) atomicExch(F.err, 2);
}

#ifndef LEANOT_SR_P
#define LEANOT_SR_P 4
#endif
#ifndef LEANOT_SR_D
#define LEANOT_SR_D 3
#endif

// LEANOT_SR=1 makes the single-read sweep the default for eligible plans.  It is opt-in: at
// n = 1e5 it measures 40.3 ms per iteration against 36.8 ms for the two-pass sweep
// (profiles/r02_single_read.md: the 148-way exchange of row partials through L2 takes
// ~1-1.5 us under full HBM load, more than the ~12 rows of exps the register file can hold
// while it is in flight; engine.sweep(single_read=True) / LEANOT_SWEEP_SINGLE_READ force it)
static bool sr_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LEANOT_SR");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// minimum n for the single-read sweep (below it the two-pass sweep's C reads hit L2)
static int64_t sr_min_n() {
  static int64_t v = -1;
  if (v < 0) {
    const char* e = getenv("LEANOT_SR_MIN_N");
    v = e ? atoll(e) : 32768;
  }
  return v;
}

// debug trace buffer (leanot_debug_sr_trace): 2 x 8 x 4096 u64 stamps, null in production
static unsigned long long* g_sr_trace = nullptr;

// workspace doubles the single-read sweep carves from plan.slab
static int64_t sr_ws_doubles(int G) { return (int64_t)SR_NSLOT * G * 2 * LEANOT_SR_P + 2; }

// Launch the single-read sweep for a plain DXG iteration if the plan qualifies (stored
// cost on the TMA path, n >= sr_min_n(), column tile <= 704, slab large enough);
// LEANOT_EINVAL: the caller runs the two-pass sweep.
static int try_sr_sweep(const leanot_dxg_plan_t& P, cudaStream_t st, bool force = false) {
  constexpr int SP = LEANOT_SR_P, SD = LEANOT_SR_D;
  using Lay = SrLayout<SP>;
  const CostView cv = make_view(P.cost);
  if (!tma_ok(cv) || (!force && (!sr_enabled() || P.n < sr_min_n()))) return LEANOT_EINVAL;
  const int G = num_sms();
  if (G > 4 * SR_CPC) return LEANOT_EINVAL;
  const int64_t W = (((P.n + G - 1) / G) + 1) & ~int64_t(1);
  if (W > SR_WMAX) return LEANOT_EINVAL;
  if (sr_ws_doubles(G) > (int64_t)P.splits * 2 * P.n) return LEANOT_EINVAL;
  auto kern = g_sr_trace ? sr_sweep_kernel<SP, SD, true> : sr_sweep_kernel<SP, SD, false>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(sr_sweep_kernel<SP, SD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Lay::SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(sr_sweep_kernel<SP, SD, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Lay::SMEM) != cudaSuccess)
      return LEANOT_EINVAL;
    if (cudaFuncSetAttribute(fused_fix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TAB_BYTES) != cudaSuccess)
      return LEANOT_EINVAL;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, SR_ALL, Lay::SMEM) != cudaSuccess || occ < 1)
      return LEANOT_EINVAL;
    attr = true;
  }
  SrArgs F;
  memset(&F, 0, sizeof(F));
  F.cost = cv;
  F.i0 = P.row0; F.i1 = P.row1;
  F.a = P.scal;
  F.b[0] = P.b; F.b[1] = P.b_bar;
  F.rw = P.r;
  F.shift = P.shift; F.m_used = P.m; F.S = P.S; F.coef = P.coef;
  F.flags = P.flags; F.col = P.col;
  F.part = reinterpret_cast<unsigned long long*>(P.slab);
  F.err = reinterpret_cast<int32_t*>(P.slab + sr_ws_doubles(G) - 2);
  F.W = W;
  F.trace = g_sr_trace;
  // generation-0 slots must read as "not ready": sign bit set (0xff bytes), error flag 0
  cudaMemsetAsync(F.part, 0xff, (size_t)(sr_ws_doubles(G) - 2) * 8, st);
  cudaMemsetAsync(F.err, 0, 16, st);
  cudaLaunchConfig_t lc;
  memset(&lc, 0, sizeof(lc));
  lc.gridDim = dim3(G);
  lc.blockDim = dim3(SR_ALL);
  lc.dynamicSmemBytes = Lay::SMEM;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&lc, kern, F);
  if (e != cudaSuccess) {
    set_error("single-read sweep launch: %s", cudaGetErrorString(e));
    return LEANOT_ECUDA;
  }
  // flagged rows: exact recompute + their column contributions (FusedArgs view of the same buffers)
  FusedArgs X;
  memset(&X, 0, sizeof(X));
  X.cost = cv; X.i0 = P.row0; X.i1 = P.row1; X.a = P.scal; X.b[0] = P.b; X.b[1] = P.b_bar; X.rw = P.r;
  X.shift = P.shift; X.m_used = P.m; X.S = P.S; X.coef = P.coef; X.flags = P.flags; X.col = P.col;
  fused_fix_kernel<<<1, 1024, TAB_BYTES, st>>>(X);
  return LEANOT_OK;
}

}  // namespace leanot

extern "C" int leanot_debug_sr_trace(void* buf) {
  leanot::g_sr_trace = reinterpret_cast<unsigned long long*>(buf);
  return LEANOT_OK;
}
