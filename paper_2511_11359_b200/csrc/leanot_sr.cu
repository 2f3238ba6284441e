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
// Variants (template parameters, LEANOT_SR_VAR): the default 'g' splits the CTAs into NG = 2
// row groups of G / 2 (each group sweeps every other panel over column tiles twice as wide,
// P = 2 rows x 2 column pairs per thread, so a row's sum is exchanged among 74 CTAs, not 148),
// parks the exps of the panels in flight in TMEM (tcgen05.st/ld, D = 5 panels) and lets the
// collector read the group's partials by cp.async into shared-memory buffers with several
// panels in flight; the groups' column sums are added in group order after the launch.
// Measured: all variants take ~37 ms per n = 1e5 iteration and 32 ms even
// with the exchange and the C copies disabled (LEANOT_SR_DBG_NOWAIT, debug timing only):
// the consumer instruction stream, not the exchange, is what binds.
// Included by leanot_lib.cu after leanot_fused.cu (mbarrier / bulk-copy helpers).

#include <type_traits>

namespace leanot {

constexpr int SR_CW = 11;                    // consumer warps
constexpr int SR_THREADS = SR_CW * 32;       // 352 consumer threads, 2 columns each
constexpr int SR_COLL = SR_THREADS;          // collector warp
constexpr int SR_NS = 6;                     // C ring slots (one panel each; 4 left ~6 % C-data waits at full HBM load)
constexpr int SR_NSLOT = 16;                 // partial-sum slots in flight (>= 2 D)
constexpr int SR_CPC = 40;                   // max CTAs per collector chunk (G <= 4 x 40)
constexpr int SR_NR = 8;                     // per-warp row-sum buffers in flight (>= D + 1)
constexpr uint64_t SR_TIMEOUT_NS = 4000000000ull;
constexpr int SR_CNB = 8;                    // async collector (row groups): partial-sum buffers in smem
#ifndef LEANOT_SR_FOLD_IN
#define LEANOT_SR_FOLD_IN 0   // 1: fold panel p - D + 1 inside panel p's exp block (measured slower: 39.6 vs 37.8 ms)
#endif
constexpr bool SR_FOLD_IN = LEANOT_SR_FOLD_IN != 0;
#ifndef LEANOT_SR_LEAD
#define LEANOT_SR_LEAD 3
#endif
constexpr int SR_LEAD = LEANOT_SR_LEAD;      // async collector: panels whose loads are in flight (< D - 1: issued after their publication)

template <int P, int NPR, int CW = SR_CW>
struct SrLayout {
  static constexpr int NV = 2 * P;                      // (row, set) partials per panel
  static constexpr int ROWB = NPR * 2 * CW * 32 * 8;    // bytes per staged row
  static constexpr int HDR = 64;                        // shift values of the panel (P <= 8)
  static constexpr int SLOT = HDR + P * ROWB;
  static constexpr int RING = TAB_BYTES;                // ring after the exp table
  static constexpr int RED = RING + SR_NS * SLOT;       // [SR_NR][CW][NV] doubles
  static constexpr int WB = RED + SR_NR * CW * NV * 8;  // [D][NV] doubles + [D][NV + 1] ints (<= 8 D)
  static constexpr int BAR = WB + 8 * (NV * 8 + (NV + 1) * 4 + 8);  // mbarriers (up to 8 D slots)
  static constexpr int CB = BAR + 8 * (2 * SR_NS + 16) + 16;   // async collector: [SR_CNB][K NV] doubles + SR_CNB mbarriers
  static constexpr int SMEM = CB;
  static constexpr int SMEM_ACOL = CB + SR_CNB * (4 * SR_CPC / 2) * 4 * 8 + SR_CNB * 8;   // K NV <= 320
  static_assert(P <= 4 && (32 % NV) == 0 && P * NPR <= 4 && ROWB % 16 == 0, "SR panel shape (collector buffers hold 2P <= 8 values per CTA)");
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
  double* gcol;           // NG > 1: NG x 2 x n column sums per row group (reduced in group order after the launch)
  unsigned long long* part;  // SR_NSLOT x G x NV tagged partials (0xff-filled before the launch)
  int32_t* err;
  int64_t W;              // column tile width (even)
  unsigned long long* trace;  // debug (null in production): per-panel timestamps of CTAs 0 and G-1
  int dbg_nowait;         // debug timing only (LEANOT_SR_DBG_NOWAIT=1): consumers do not wait for g, no collector
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


// ---- TMEM parking of the exps (TM variant) ----
// A consumer warp may touch only its lane quarter of TMEM (lanes 32 (warp % 4) ..); the
// 32x32b shape gives each thread one lane, so a thread parks its 16 doubles of a panel as 32
// consecutive 32-bit columns of its own lane.
#define SR_R32(a) "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]), \
  "r"(a[8]), "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]), "r"(a[15]), "r"(a[16]), \
  "r"(a[17]), "r"(a[18]), "r"(a[19]), "r"(a[20]), "r"(a[21]), "r"(a[22]), "r"(a[23]), "r"(a[24]), "r"(a[25]), \
  "r"(a[26]), "r"(a[27]), "r"(a[28]), "r"(a[29]), "r"(a[30]), "r"(a[31])
#define SR_W32(a) "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7]), \
  "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]), "=r"(a[14]), "=r"(a[15]), \
  "=r"(a[16]), "=r"(a[17]), "=r"(a[18]), "=r"(a[19]), "=r"(a[20]), "=r"(a[21]), "=r"(a[22]), "=r"(a[23]), \
  "=r"(a[24]), "=r"(a[25]), "=r"(a[26]), "=r"(a[27]), "=r"(a[28]), "=r"(a[29]), "=r"(a[30]), "=r"(a[31])
#define SR_RW32(a) "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]), \
  "+r"(a[8]), "+r"(a[9]), "+r"(a[10]), "+r"(a[11]), "+r"(a[12]), "+r"(a[13]), "+r"(a[14]), "+r"(a[15]), \
  "+r"(a[16]), "+r"(a[17]), "+r"(a[18]), "+r"(a[19]), "+r"(a[20]), "+r"(a[21]), "+r"(a[22]), "+r"(a[23]), \
  "+r"(a[24]), "+r"(a[25]), "+r"(a[26]), "+r"(a[27]), "+r"(a[28]), "+r"(a[29]), "+r"(a[30]), "+r"(a[31])

__device__ __forceinline__ void sr_tm_st(uint32_t ta, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(ta), SR_R32(v) : "memory");
}
__device__ __forceinline__ void sr_tm_ld(uint32_t ta, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : SR_W32(v) : "r"(ta) : "memory");
}
// wait for this thread's TMEM loads; the loaded registers are tied to the wait so no use of
// them can be scheduled above it
__device__ __forceinline__ void sr_tm_wait_ld(uint32_t (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : SR_RW32(v) :: "memory");
}
// 24-word forms (12 doubles per thread and panel): x16 + x8
__device__ __forceinline__ void sr_tm_st24(uint32_t ta, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               ::"r"(ta + 16), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]),
               "r"(v[23]) : "memory");
}
__device__ __forceinline__ void sr_tm_ld24(uint32_t ta, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]) : "r"(ta) : "memory");
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23])
               : "r"(ta + 16) : "memory");
}

// 16 doubles per thread as 32 TMEM columns, the 64-bit halves split / joined inside the asm so
// the compiler keeps the doubles in their register pairs (no moves); the load waits for its
// own completion before the joins
__device__ __forceinline__ void sr_tm_st16d(uint32_t ta, const double (&e)[16]) {
  asm volatile("{\n\t.reg .b32 t<32>;\n\t"
      "mov.b64 {t0, t1}, %1;\n\t""mov.b64 {t2, t3}, %2;\n\t""mov.b64 {t4, t5}, %3;\n\t""mov.b64 {t6, t7}, %4;\n\t""mov.b64 {t8, t9}, %5;\n\t""mov.b64 {t10, t11}, %6;\n\t""mov.b64 {t12, t13}, %7;\n\t""mov.b64 {t14, t15}, %8;\n\t""mov.b64 {t16, t17}, %9;\n\t""mov.b64 {t18, t19}, %10;\n\t""mov.b64 {t20, t21}, %11;\n\t""mov.b64 {t22, t23}, %12;\n\t""mov.b64 {t24, t25}, %13;\n\t""mov.b64 {t26, t27}, %14;\n\t""mov.b64 {t28, t29}, %15;\n\t""mov.b64 {t30, t31}, %16;\n\t"
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {t0, t1, t2, t3, t4, t5, t6, t7, t8, t9, t10, t11, t12, t13, t14, t15, t16, t17, t18, t19, t20, t21, t22, t23, t24, t25, t26, t27, t28, t29, t30, t31};\n\t}"
      ::"r"(ta), "d"(e[0]), "d"(e[1]), "d"(e[2]), "d"(e[3]), "d"(e[4]), "d"(e[5]), "d"(e[6]), "d"(e[7]), "d"(e[8]), "d"(e[9]), "d"(e[10]), "d"(e[11]), "d"(e[12]), "d"(e[13]), "d"(e[14]), "d"(e[15]) : "memory");
}
__device__ __forceinline__ void sr_tm_ld16d(uint32_t ta, double (&e)[16]) {
  asm volatile("{\n\t.reg .b32 t<32>;\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {t0, t1, t2, t3, t4, t5, t6, t7, t8, t9, t10, t11, t12, t13, t14, t15, t16, t17, t18, t19, t20, t21, t22, t23, t24, t25, t26, t27, t28, t29, t30, t31}, [%16];\n\t"
      "tcgen05.wait::ld.sync.aligned;\n\t"
      "mov.b64 %0, {t0, t1};\n\t""mov.b64 %1, {t2, t3};\n\t""mov.b64 %2, {t4, t5};\n\t""mov.b64 %3, {t6, t7};\n\t""mov.b64 %4, {t8, t9};\n\t""mov.b64 %5, {t10, t11};\n\t""mov.b64 %6, {t12, t13};\n\t""mov.b64 %7, {t14, t15};\n\t""mov.b64 %8, {t16, t17};\n\t""mov.b64 %9, {t18, t19};\n\t""mov.b64 %10, {t20, t21};\n\t""mov.b64 %11, {t22, t23};\n\t""mov.b64 %12, {t24, t25};\n\t""mov.b64 %13, {t26, t27};\n\t""mov.b64 %14, {t28, t29};\n\t""mov.b64 %15, {t30, t31};\n\t"
      "}"
      : "=d"(e[0]), "=d"(e[1]), "=d"(e[2]), "=d"(e[3]), "=d"(e[4]), "=d"(e[5]), "=d"(e[6]), "=d"(e[7]), "=d"(e[8]), "=d"(e[9]), "=d"(e[10]), "=d"(e[11]), "=d"(e[12]), "=d"(e[13]), "=d"(e[14]), "=d"(e[15]) : "r"(ta) : "memory");
}
__device__ __forceinline__ void sr_tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <int P, int D, bool TRACE, bool TM, int NG, int NPR, bool ACOL, int CW>
__global__ void __launch_bounds__(CW * 32 + 32, 1) sr_sweep_kernel(const SrArgs F) {
  using L = SrLayout<P, NPR, CW>;
  constexpr int NV = L::NV;
  constexpr int THREADS = CW * 32, COLL = THREADS;   // consumer threads; the collector warp follows
  constexpr int NE = P * NPR * 4;   // exps per thread and panel (rows x pairs x sets x 2 columns)
  constexpr int SW = 2 * NE;        // TMEM columns per parked panel
  static_assert(!TM || NE == 16 || NE == 12, "TMEM slot = 32 or 24 columns");
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
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_cnt + SR_NR);     // TMEM base address (TM)
  static_assert(SR_NS + 2 * D + 1 + SR_NR / 2 + 1 <= 2 * SR_NS + 16 && SR_NR >= D + 1 && 2 * D <= SR_NSLOT, "SR slots");
  // TM: up to (CW + 3) / 4 consumer warps share a lane quarter, each parks D panels x SW columns
  static_assert(!TM || ((CW + 3) / 4) * SW * D <= 512, "TMEM slots");
  load_table(reinterpret_cast<double*>(smem));
  if (threadIdx.x == 0) {
    for (int s = 0; s < SR_NS; ++s) mbar_init(full + s, 1);
    for (int s = 0; s < D; ++s) { mbar_init(wready + s, 1); mbar_init(wfree + s, CW); }
    *s_abort = 0;
    for (int i = 0; i < SR_NR; ++i) s_cnt[i] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (TM && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = TM ? *reinterpret_cast<volatile uint32_t*>(s_tmem) : 0u;

  const CostView& cv = F.cost;
  const int64_t n = cv.n, nr = F.i1 - F.i0;
  const int64_t npan = (nr + P - 1) / P;                 // panels of the sweep
  const int G = gridDim.x, c = blockIdx.x;
  const int K = G / NG, grp = c / K, kc = c - grp * K;  // row group of this CTA and its rank in it
  // group grp takes panels q = t NG + grp, t = 0 .. npl - 1
  const int npl = (int)(npan > grp ? (npan - grp + NG - 1) / NG : 0);
  const int64_t j0 = (int64_t)kc * F.W, j1 = j0 + F.W < n ? j0 + F.W : n;
  const uint32_t wbytes = j0 < j1 ? (uint32_t)((j1 - j0) * 8) : 0u;
  const int lane = threadIdx.x & 31;
  unsigned long long* trace =
      TRACE && F.trace && (c == 0 || c == G - 1) ? F.trace + (c == 0 ? 0 : 8 * 4096) : nullptr;
  if (!TRACE || npl > 4096) trace = nullptr;

  if (threadIdx.x >= COLL && F.dbg_nowait) return;
  if (threadIdx.x >= COLL) {  // ------------------------- collector warp -------------------------
    // Layout of a panel's partials: [CTA c][v = 2 r + k], the group's K CTAs contiguous.  Lane
    // l loads 16-byte pairs at doubles 2 l + 64 jj: values v0 = 2 (l % LPC), v0 + 1 of CTA
    // CPL jj + l / LPC (LPC = NV / 2 lanes per CTA), so lanes l ^ LPC, l ^ 2 LPC, ... hold the
    // same two values of other CTAs and butterfly levels o = LPC .. 16 finish the sums.  The
    // order (jj ascending per lane, then the butterfly) is fixed, so every CTA of the group
    // computes bitwise the same S.
    // Generation tags: a value of parity `par` carries sign bit `par`; the raw doubles are
    // summed as they are (for par = 1 every term is negated, so S = -sum exactly) and a load
    // is stale if any value's sign bit differs.
    // The loads are direct relaxed loads, all in flight at once, and software-pipelined:
    // panel t + 1's loads are issued before panel t's S are finalized.
    constexpr int LPC = NV / 2, CPL = 32 / LPC;
    constexpr int NJ = (4 * SR_CPC / NG * NV + 63) / 64;   // 16-byte loads per lane covering K <= 160 / NG
    const int cl = lane / LPC;
    const int njj = (K + CPL - 1) / CPL;
    bool dead = false;
    double2 y[NJ];
    auto issue = [&](int t) {
      const double2* gp = reinterpret_cast<const double2*>(F.part + ((t % SR_NSLOT) * G + grp * K) * NV) + lane;
#pragma unroll
      for (int jj = 0; jj < NJ; ++jj)
        if (jj < njj && CPL * jj + cl < K) {
          unsigned long long u0, u1;
          asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(u0), "=l"(u1) : "l"(gp + 32 * jj));
          y[jj] = make_double2(__longlong_as_double((long long)u0), __longlong_as_double((long long)u1));
        }
    };
    // ACOL: the group's partials of panel t arrive by cp.async (L2, 16 bytes per lane) in smem
    // buffer t % SR_CNB, completion on that buffer's mbarrier (32 lane arrivals per issue);
    // loads of the next SR_LEAD panels are in flight while panel t is finalized, so the
    // collector is not limited to one L2 round trip per panel
    static_assert(!ACOL || NG >= 2, "async collector buffers are sized for row groups");
    constexpr int KNV = (4 * SR_CPC / NG) * NV;                // buffer doubles (K <= 160 / NG)
    double* cb = reinterpret_cast<double*>(smem + L::CB);
    uint64_t* cbar = reinterpret_cast<uint64_t*>(smem + L::CB + SR_CNB * KNV * 8);
    uint32_t cph = 0;                                           // wait parity per buffer
    auto aissue = [&](int t) {
      const int bi = t % SR_CNB;
      const char* src = reinterpret_cast<const char*>(F.part + ((t % SR_NSLOT) * G + grp * K) * NV);
      const uint32_t dst = smem_u32(cb + bi * KNV);
#pragma unroll
      for (int jj = 0; jj < NJ; ++jj)
        if (jj < njj && CPL * jj + cl < K)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * (lane + 32 * jj)),
                       "l"(src + 16 * (lane + 32 * jj)) : "memory");
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(cbar + bi)) : "memory");
    };
    if (ACOL) {
      if (lane == 0)
        for (int i = 0; i < SR_CNB; ++i) mbar_init(cbar + i, 32);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      __syncwarp();
      for (int u = 0; u < SR_LEAD && u < npl; ++u) aissue(u);
    } else if (npl > 0) {
      issue(0);
    }
    // lanes 0 .. P-1 finalize row r = lane of each panel: r_i prefetched one panel ahead
    auto row_of = [&](int t) { return ((int64_t)t * NG + grp) * P + lane; };
    double rw_next = (lane < P && npl > 0 && row_of(0) < nr) ? __ldg(F.rw + F.i0 + row_of(0)) : 0.0;
    for (int t = 0; t < npl; ++t) {
      const unsigned long long parbits = (unsigned long long)((t / SR_NSLOT) & 1) << 63;
      const double rw_q = rw_next;
      if (t + 1 < npl && lane < P) {
        const int64_t li1 = row_of(t + 1);
        rw_next = li1 < nr ? __ldg(F.rw + F.i0 + li1) : 0.0;
      }
      if (TRACE && trace && lane == 0) trace[t * 8 + 1] = clock64();
      double a0, a1, c0, c1;   // (v0, v1) x (even jj, odd jj)
      const uint64_t t0 = sr_now();
      int rounds = 0;
      while (true) {
        if (ACOL) {   // wait for this panel's buffer, then read it
          const int bi = t % SR_CNB;
          sr_wait(cbar + bi, (cph >> bi) & 1u, s_abort);
          cph ^= 1u << bi;
          const double2* bp = reinterpret_cast<const double2*>(cb + bi * KNV) + lane;
#pragma unroll
          for (int jj = 0; jj < NJ; ++jj)
            if (jj < njj && CPL * jj + cl < K) y[jj] = bp[32 * jj];
        }
        a0 = a1 = c0 = c1 = 0.0;
        const unsigned p32 = (unsigned)(parbits >> 32);
        unsigned bad = 0;
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj)
          if (jj < njj && CPL * jj + cl < K) {
            bad |= ((unsigned)__double2hiint(y[jj].x) ^ p32);
            bad |= ((unsigned)__double2hiint(y[jj].y) ^ p32);
            if (jj & 1) { c0 += y[jj].x; c1 += y[jj].y; } else { a0 += y[jj].x; a1 += y[jj].y; }
          }
        if (!__any_sync(0xffffffffu, bad >> 31) || dead) break;
        ++rounds;
        const uint64_t el = sr_now() - t0;
        if (__any_sync(0xffffffffu, el > SR_TIMEOUT_NS || (el > 1000000ull && *(volatile int32_t*)F.err != 0))) {
          dead = true;   // co-residency / protocol failure (never expected): report and drain
          if (lane == 0) atomicExch(F.err, 1);
          break;
        }
        if (ACOL) {
          __syncwarp();
          aissue(t);
        } else {
          issue(t);
        }
      }
      if (ACOL) {
        __syncwarp();   // every lane has read buffer t % SR_CNB before any reuse
        if (t + SR_LEAD < npl) aissue(t + SR_LEAD);
      } else if (t + 1 < npl) {
        issue(t + 1);   // next panel's round trip overlaps this finalization
      }
      if (TRACE && trace && lane == 0) { trace[t * 8 + 2] = clock64(); trace[t * 8 + 7] = rounds; }
      double s0 = a0 + c0, s1 = a1 + c1;
#pragma unroll
      for (int o = LPC; o < 32; o <<= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      }
      if (parbits) { s0 = -s0; s1 = -s1; }
      if (TRACE && trace && lane == 0) trace[t * 8 + 3] = clock64();
      // lanes 0..P-1: row r = lane, S0 = S of the current weights, S1 = S of the midpoint weights
      const int64_t li = row_of(t);
      const bool valid = lane < P && li < nr;
      const bool ok0 = valid && sum_ok(s0) && !dead, ok1 = valid && sum_ok(s1) && !dead;
      // g = r_i / S: one correctly rounded reciprocal and a multiply (<= 1.5 ulp of the quotient)
      const double w0 = ok0 ? rw_q * __drcp_rn(s0) : 0.0, w1 = ok1 ? rw_q * __drcp_rn(s1) : 0.0;
      const int ds = t % D;
      if (t >= D) sr_wait(wfree + ds, (uint32_t)(((t / D) - 1) & 1), s_abort);
      if (lane < P) {
        wbuf[ds * NV + 2 * lane] = w0;
        wbuf[ds * NV + 2 * lane + 1] = w1;
        okbuf[ds * (NV + 1) + 2 * lane] = ok0 ? 1 : 0;
        okbuf[ds * (NV + 1) + 2 * lane + 1] = ok1 ? 1 : 0;
      }
      const bool all = __all_sync(0xffffffffu, lane >= P || (ok0 && ok1));
      if (lane == 0) okbuf[ds * (NV + 1) + NV] = all ? 1 : 0;
      __syncwarp();
      if (TRACE && trace && lane == 0) trace[t * 8 + 4] = clock64();
      if (lane == 0) mbar_arrive(wready + ds);
      if (valid && t % K == kc) {  // one CTA of the group finalizes the panel's rows (off the consumers' path)
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
  // SMSP 3 with warps 3 and 7, so warp 7 takes the LAST column group, which is the least
  // filled when W < NPR x 704, leaving the collector issue slots.
  constexpr int WS = CW - 4;   // last consumer warp on the collector's SMSP
  const int cgrp = warp == WS ? CW - 1 : (warp == CW - 1 ? WS : warp);
  const int tcol = cgrp * 32 + lane;
  // column pair u of this thread: local columns jt[u], jt[u] + 1 (n and W even: pairs are whole)
  int jt[NPR];
  bool has[NPR];
  double na[2], nb[2][NPR][2], acc[2][NPR][2];
#pragma unroll
  for (int u = 0; u < NPR; ++u) {
    jt[u] = 2 * tcol + 2 * THREADS * u;
    has[u] = j0 + jt[u] < j1;
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    na[k] = -F.a[k];
#pragma unroll
    for (int u = 0; u < NPR; ++u) {
      nb[k][u][0] = has[u] ? -__ldg(F.b[k] + j0 + jt[u]) : 0.0;
      nb[k][u][1] = has[u] ? -__ldg(F.b[k] + j0 + jt[u] + 1) : 0.0;
      acc[k][u][0] = 0.0; acc[k][u][1] = 0.0;
    }
  }
  uint32_t s = 0, ph = 0;
  // thread 0: fill ring slot `slot` with local panel t (row shifts + the C tile rows)
  auto refill = [&](int t, int slot) {
    const int64_t li0 = ((int64_t)t * NG + grp) * P;
    const int rows = (int)(nr - li0 < P ? nr - li0 : P);
    char* dst = ring + slot * L::SLOT;
    uint64_t* bar = full + slot;
    if (F.dbg_nowait == 2) {   // debug timing: no C data (the slot keeps stale contents)
      mbar_arrive(bar);
      return;
    }
    if (rows < P || P * 8 < 16) {  // last, partial panel (a bulk copy would read past nr) or a
                                   // header below the bulk copy's 16-byte minimum: plain loads
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
    for (int q = 0; q < SR_NS && q < npl; ++q) refill(q, q);
  // running panel bookkeeping (32-bit, no divisions in the loop): reduction buffer pr = p % NR,
  // partial-sum slot ps = p % NSLOT with generation parity pp
  int pr = 0, ps = 0;
  unsigned long long pp = 0;
  // warps whose every lane has all its column pairs (all but the tail warps) skip the
  // per-pair selects; both forms add the same terms in the same order
  bool allhas = true;
#pragma unroll
  for (int u = 0; u < NPR; ++u) allhas = allhas && has[u];
  const bool warp_full = __all_sync(0xffffffffu, allhas);
  auto compute_f = [&](int p, double (&E)[P][NPR][2][2], auto fullc, const double (*Eq)[NPR][2][2],
                       const double* gq) {
    constexpr bool fw = decltype(fullc)::value;
    sr_wait(full + s, ph, s_abort);
    const char* st = ring + s * L::SLOT;
    double rs[NV];
    {
      // threads without columns (the last CTA's tail) compute on column pair 0 of the slot and
      // contribute 0 to the row sums: no divergent zero-filling of the exps (their column sums
      // are never written)
      const uint32_t* hdr = reinterpret_cast<const uint32_t*>(st);  // int64 shifts: low words at 2r
#pragma unroll
      for (int r = 0; r < P; ++r) {
        const uint32_t ml = hdr[2 * r];
        rs[r * 2] = 0.0;
        rs[r * 2 + 1] = 0.0;
#pragma unroll
        for (int u = 0; u < NPR; ++u) {
          const int tc = has[u] ? jt[u] : 0;
          const double2 cc = *reinterpret_cast<const double2*>(st + L::HDR + r * L::ROWB + 8 * tc);
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            E[r][u][k][0] = texp(tb, fma(na[k], cc.x, nb[k][u][0]), ml);
            E[r][u][k][1] = texp(tb, fma(na[k], cc.y, nb[k][u][1]), ml);
            rs[r * 2 + k] += (fw || has[u]) ? E[r][u][k][0] + E[r][u][k][1] : 0.0;
          }
        }
      }
      if (Eq) {   // fold of an earlier panel (every row ok), scheduled among this panel's exps
#pragma unroll
        for (int r = 0; r < P; ++r)
#pragma unroll
          for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int u = 0; u < NPR; ++u) {
              acc[k][u][0] = fma(gq[r * 2 + k], Eq[r][u][k][0], acc[k][u][0]);
              acc[k][u][1] = fma(gq[r * 2 + k], Eq[r][u][k][1], acc[k][u][1]);
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
    double* rb = red + pr * (CW * NV);
    if ((lane & (32 / NV - 1)) == 0) rb[warp * NV + lane / (32 / NV)] = y;
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      __threadfence_block();
      last = atomicAdd(s_cnt + pr, 1) == CW - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      __threadfence_block();
      if (lane == 0) {
        s_cnt[pr] = 0;   // reused NR panels later, after this CTA's partial of p + 1 is out
        if (p + SR_NS < npl) refill(p + SR_NS, used);
      }
      if (lane < NV) {
        const volatile double* vb = rb;
        double t = vb[lane];
#pragma unroll
        for (int w = 1; w < CW; ++w) t += vb[w * NV + lane];
        const unsigned long long bits = ((unsigned long long)__double_as_longlong(t) & 0x7fffffffffffffffull) | pp;
        st_relaxed_u64(F.part + (ps * G + c) * NV + lane, bits);
        if (TRACE && trace && lane == 0) trace[p * 8] = clock64();
      }
    }
    if (++pr == SR_NR) pr = 0;
    if (++ps == SR_NSLOT) { ps = 0; pp ^= 1ull << 63; }
  };
  auto compute = [&](int p, double (&E)[P][NPR][2][2]) {
    if (warp_full) compute_f(p, E, std::true_type{}, nullptr, nullptr);
    else compute_f(p, E, std::false_type{}, nullptr, nullptr);
  };
  auto compute_fold = [&](int p, double (&E)[P][NPR][2][2], const double (&Eq)[P][NPR][2][2], const double* gq) {
    if (warp_full) compute_f(p, E, std::true_type{}, Eq, gq);
    else compute_f(p, E, std::false_type{}, Eq, gq);
  };
  // fold panel q (exps E, slot ds = q % D, wready parity wpar) into the column sums
  auto accumulate = [&](int q, const double (&E)[P][NPR][2][2], int ds, uint32_t wpar) {
    if (TRACE && trace && threadIdx.x == 0) trace[q * 8 + 5] = clock64();
    if (!F.dbg_nowait) sr_wait(wready + ds, wpar, s_abort);
    if (TRACE && trace && threadIdx.x == 0) trace[q * 8 + 6] = clock64();
    const double* wq = wbuf + ds * NV;
    const int* oq = okbuf + ds * (NV + 1);
    if (oq[NV]) {
#pragma unroll
      for (int r = 0; r < P; ++r)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const double g = wq[r * 2 + k];
#pragma unroll
          for (int u = 0; u < NPR; ++u) {
            acc[k][u][0] = fma(g, E[r][u][k][0], acc[k][u][0]);
            acc[k][u][1] = fma(g, E[r][u][k][1], acc[k][u][1]);
          }
        }
    } else {
#pragma unroll
      for (int r = 0; r < P; ++r)
#pragma unroll
        for (int k = 0; k < 2; ++k)
          if (oq[r * 2 + k]) {
            const double g = wq[r * 2 + k];
#pragma unroll
            for (int u = 0; u < NPR; ++u) {
              acc[k][u][0] = fma(g, E[r][u][k][0], acc[k][u][0]);
              acc[k][u][1] = fma(g, E[r][u][k][1], acc[k][u][1]);
            }
          }
    }
    release(wfree + ds);
  };
  if constexpr (TM) {
    // exps parked in TMEM: panel p is computed in registers, stored to slot p % D, and
    // reloaded for the fold D - 1 panels later (the load is issued before the next compute)
    const uint32_t tw = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * SW * D);
    double E[P][NPR][2][2];
    uint32_t Fv[32];
    for (int p = 0; p < npl + D - 1; ++p) {
      const int q = p - (D - 1);
      sr_tm_wait_st();   // the previous panel's store (q <= p - 2 was stored before it)
      if constexpr (NE != 16) {
        if (q >= 0) sr_tm_ld24(tw + SW * (q % D), Fv);
      }
      bool folded = false;
      if constexpr (NE == 16 && SR_FOLD_IN) {
        if (q >= 0 && p < npl) {
          // wait for g of panel q first, then compute panel p with q's fold in the same block
          const int ds = q % D;
          if (!F.dbg_nowait) sr_wait(wready + ds, (uint32_t)((q / D) & 1), s_abort);
          const int* oq = okbuf + ds * (NV + 1);
          if (oq[NV]) {
            double Eq[P][NPR][2][2];
            sr_tm_ld16d(tw + SW * (q % D), reinterpret_cast<double(&)[16]>(Eq));
            double gq[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) gq[v] = wbuf[ds * NV + v];
            compute_fold(p, E, Eq, gq);
            release(wfree + ds);
            folded = true;
          }
        }
      }
      if (p < npl) {
        if (!folded) compute(p, E);
        if constexpr (NE == 16) {
          sr_tm_st16d(tw + SW * (p % D), reinterpret_cast<const double(&)[16]>(E));
        } else {
          uint32_t ev[32];
          const double* Ef = &E[0][0][0][0];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            ev[2 * i] = i < NE ? (uint32_t)__double2loint(Ef[i]) : 0u;
            ev[2 * i + 1] = i < NE ? (uint32_t)__double2hiint(Ef[i]) : 0u;
          }
          sr_tm_st24(tw + SW * (p % D), ev);
        }
      }
      if (q >= 0 && !folded) {
        double Eq[P][NPR][2][2];
        if constexpr (NE == 16) {
          sr_tm_ld16d(tw + SW * (q % D), reinterpret_cast<double(&)[16]>(Eq));
        } else {
          sr_tm_wait_ld(Fv);
          double* Ef = &Eq[0][0][0][0];
#pragma unroll
          for (int i = 0; i < NE; ++i) Ef[i] = __hiloint2double((int)Fv[2 * i + 1], (int)Fv[2 * i]);
        }
        accumulate(q, Eq, q % D, (uint32_t)((q / D) & 1));
      }
    }
  } else {
    double e[D][P][NPR][2][2];
    // p0 steps by D, so panel p = p0 + u keeps its exps in e[u] and panel q = p - (D - 1) is in
    // e[(u + 1) % D] with wready slot (u + 1) % D; its use index q / D is p0 / D for u = D - 1
    // and p0 / D - 1 otherwise (phase bit wph tracks p0 / D)
    uint32_t wph = 0;
    for (int p0 = 0; p0 < npl + D - 1; p0 += D, wph ^= 1) {
#pragma unroll
      for (int u = 0; u < D; ++u) {
        const int p = p0 + u;
        if (p < npl) compute(p, e[u]);
        const int q = p - (D - 1);
        if (q >= 0 && q < npl) accumulate(q, e[(u + 1) % D], (u + 1) % D, u == D - 1 ? wph : wph ^ 1);
      }
    }
  }
  // column sums of this group's rows: directly into col (one group) or into the group's slab
  double* out = NG == 1 ? F.col : F.gcol + (int64_t)grp * 2 * n;
#pragma unroll
  for (int u = 0; u < NPR; ++u)
    if (has[u]) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        out[k * n + j0 + jt[u]] = acc[k][u][0];
        out[k * n + j0 + jt[u] + 1] = acc[k][u][1];
      }
    }
  if (TM) {   // consumers only (the collector has returned): free TMEM after every warp's last load
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"n"(THREADS) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
  if (*s_abort && threadIdx.x == 0) atomicExch(F.err, 2);
}

// Variants (LEANOT_SR_VAR): 'g' (default) row groups: NG = 2 groups of G / 2 CTAs, each
// group sweeps every other panel of P = 2 rows over column tiles of W <= 1408 (2 column pairs
// per thread), exps parked in TMEM for D = 5 panels, the two groups' column sums reduced in
// group order after the launch; 't': one group, P = 4 rows, 1 pair per thread, TMEM (D = 5);
// 'r': one group, exps in registers (D = 3).
static char sr_variant() {
  static char v = 0;
  if (!v) {
    const char* e = getenv("LEANOT_SR_VAR");
    v = (e && (e[0] == 't' || e[0] == 'r' || e[0] == 'h' || e[0] == 'w')) ? e[0] : 'g';
  }
  return v;
}

// LEANOT_SR=1 makes the single-read sweep the default for eligible plans (engine.sweep(
// single_read=True) / LEANOT_SWEEP_SINGLE_READ force it).
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

// partial-sum slots + error flag the single-read sweep carves from plan.slab (NV = 8 covers
// every variant: 2 P <= 8)
static int64_t sr_ws_doubles(int G) { return (int64_t)SR_NSLOT * G * 8 + 2; }

template <int P, int D, bool TM, int NG, int NPR, bool ACOL, int CW = SR_CW>
static int launch_sr_variant(const leanot_dxg_plan_t& Pl, const CostView& cv, cudaStream_t st) {
  using Lay = SrLayout<P, NPR, CW>;
  constexpr int NT = CW * 32 + 32;
  constexpr int SMEM = ACOL ? Lay::SMEM_ACOL : Lay::SMEM;
  const int G = num_sms();
  if (G % NG != 0 || G / NG > 4 * SR_CPC / NG) return LEANOT_EINVAL;
  const int K = G / NG;
  const int64_t W = (((Pl.n + K - 1) / K) + 1) & ~int64_t(1);
  if (W > NPR * 2 * CW * 32) return LEANOT_EINVAL;
  const int64_t gcol_off = (sr_ws_doubles(G) + 15) & ~int64_t(15);
  const int64_t need = NG > 1 ? gcol_off + (int64_t)NG * 2 * Pl.n : sr_ws_doubles(G);
  if (need > (int64_t)Pl.splits * 2 * Pl.n) return LEANOT_EINVAL;
  auto kern = g_sr_trace ? sr_sweep_kernel<P, D, true, TM, NG, NPR, ACOL, CW> : sr_sweep_kernel<P, D, false, TM, NG, NPR, ACOL, CW>;
  static bool attr = false;
  if (!attr) {
    for (auto kk : {sr_sweep_kernel<P, D, true, TM, NG, NPR, ACOL, CW>, sr_sweep_kernel<P, D, false, TM, NG, NPR, ACOL, CW>})
      if (cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess)
        return LEANOT_EINVAL;
    if (cudaFuncSetAttribute(fused_fix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TAB_BYTES) != cudaSuccess)
      return LEANOT_EINVAL;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, SMEM) != cudaSuccess || occ < 1)
      return LEANOT_EINVAL;
    attr = true;
  }
  SrArgs F;
  memset(&F, 0, sizeof(F));
  F.cost = cv;
  F.i0 = Pl.row0; F.i1 = Pl.row1;
  F.a = Pl.scal;
  F.b[0] = Pl.b; F.b[1] = Pl.b_bar;
  F.rw = Pl.r;
  F.shift = Pl.shift; F.m_used = Pl.m; F.S = Pl.S; F.coef = Pl.coef;
  F.flags = Pl.flags; F.col = Pl.col;
  F.gcol = NG > 1 ? Pl.slab + gcol_off : nullptr;
  F.part = reinterpret_cast<unsigned long long*>(Pl.slab);
  F.err = reinterpret_cast<int32_t*>(Pl.slab + sr_ws_doubles(G) - 2);
  F.W = W;
  F.trace = g_sr_trace;
  {
    const char* e = getenv("LEANOT_SR_DBG_NOWAIT");
    F.dbg_nowait = e ? atoi(e) : 0;
    static bool warned = false;
    if (F.dbg_nowait && !warned) {
      fprintf(stderr, "leanot: LEANOT_SR_DBG_NOWAIT=%d -- single-read sweeps run in a timing-only debug mode "
                      "and their results are WRONG\n", F.dbg_nowait);
      warned = true;
    }
  }
  // generation-0 slots must read as "not ready": sign bit set (0xff bytes), error flag 0
  cudaMemsetAsync(F.part, 0xff, (size_t)(sr_ws_doubles(G) - 2) * 8, st);
  cudaMemsetAsync(F.err, 0, 16, st);
  cudaLaunchConfig_t lc;
  memset(&lc, 0, sizeof(lc));
  lc.gridDim = dim3(G);
  lc.blockDim = dim3(NT);
  lc.dynamicSmemBytes = SMEM;
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
  // row groups: their column sums added in group order (deterministic)
  if (NG > 1) LEANOT_TRY(launch_slab_reduce(F.gcol, NG, 2, Pl.n, Pl.col, st));
  // flagged rows: exact recompute + their column contributions (FusedArgs view of the same buffers)
  FusedArgs X;
  memset(&X, 0, sizeof(X));
  X.cost = cv; X.i0 = Pl.row0; X.i1 = Pl.row1; X.a = Pl.scal; X.b[0] = Pl.b; X.b[1] = Pl.b_bar; X.rw = Pl.r;
  X.shift = Pl.shift; X.m_used = Pl.m; X.S = Pl.S; X.coef = Pl.coef; X.flags = Pl.flags; X.col = Pl.col;
  fused_fix_kernel<<<1, 1024, TAB_BYTES, st>>>(X);
  return LEANOT_OK;
}

// Launch the single-read sweep for a plain DXG iteration if the plan qualifies (stored
// cost on the TMA path, n >= sr_min_n(), column tile within the variant's width, slab large
// enough); LEANOT_EINVAL: the caller runs the two-pass sweep.
static int try_sr_sweep(const leanot_dxg_plan_t& P, cudaStream_t st, bool force = false) {
  const CostView cv = make_view(P.cost);
  if (!tma_ok(cv) || (!force && (!sr_enabled() || P.n < sr_min_n()))) return LEANOT_EINVAL;
  const char v = sr_variant();
  if (v == 'w') {
    const int rc = launch_sr_variant<1, 5, true, 4, 3, true, 15>(P, cv, st);
    if (rc != LEANOT_EINVAL) return rc;
  }
  if (v == 'g' || v == 'h') {
    const int rc = v == 'g' ? launch_sr_variant<2, 5, true, 2, 2, true>(P, cv, st)
                            : launch_sr_variant<2, 5, true, 2, 2, false>(P, cv, st);
    if (rc != LEANOT_EINVAL) return rc;   // plans outside the grouped shape take the one-group form
  }
  if (v == 'r') return launch_sr_variant<4, 3, false, 1, 1, false>(P, cv, st);
  return launch_sr_variant<4, 5, true, 1, 1, false>(P, cv, st);
}

}  // namespace leanot

extern "C" int leanot_debug_sr_trace(void* buf) {
  leanot::g_sr_trace = reinterpret_cast<unsigned long long*>(buf);
  return LEANOT_OK;
}
