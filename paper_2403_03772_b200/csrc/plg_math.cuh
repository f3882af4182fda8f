// plg_math.cuh — FP64 element math of the entropy approximation, sm_100a.
//
// One "EDE" (element-direction evaluation) is one sample u of one residual entropy
// (reference proj/src/kernels.cpp:16-34):
//     lc  = |u| + (log1p(exp(-2|u|)) - ln2)      (log cosh u)
//     pdf = u * exp(-u^2 / 2)
// libdevice exp + log1p + exp cost ~70 FP64-pipe instructions per EDE. Here both
// exponentials use a 128-entry 2^(j/128) table (|reduced arg| <= ln2/256) and log1p a
// 128-entry reciprocal/log table (|r| <= 1/257), each finished by a degree-4 near-minimax
// polynomial (tools/fit_polys.py). Absolute error per element is a few ulp of lc and pdf
// (tests/test_gpu_parity.py checks against libdevice and numpy); the causal order needs
// ~1e-9.
//
// Throughput is bound by register-file reads rather than by the FP64 pipe itself: a DFMA
// reading 3 distinct register pairs takes 3 issue cycles instead of 2, and integer
// instructions share the read ports (measured, tools/probe/fp64_mix.cu; model and SASS
// census in tools/rf_model.py). The formulation below is shaped by that:
//   * the caller supplies u scaled by K = 256/ln2, so exp(-2|u|) reduces with one
//     immediate-operand DADD (k = rint(-|u'|), r' = |u'| + k) instead of two DFMAs with a
//     register constant; sum |u| is kept apart and rescaled once at the end;
//   * each polynomial's leading coefficient is a short double, so its first Horner step
//     is DMUL-by-immediate + DADD (1 register pair each) instead of a 3-pair DFMA;
//   * the 2^(j/128) table is pre-compensated so 2^(k/128) costs one IMAD after the row
//     load (exp2_k), and |u| is left to FP64 operand modifiers (no integer abs + move).
//   Integer instructions per EDE: 18.4 (v3) -> 12.5; FP64-pipe active 78.6% -> 82.0%.
//
// Shared-memory tables, replicated per lane group so random per-lane indices never
// bank-conflict:
//   exp: 128 rows x 16 lanes x 8 B  (row j = 2^(j/128); a half-warp reads 16 distinct banks)
//   log: 256 rows x  8 lanes x 16 B (row 128 + j = {c_j, -log(c_j) - ln2} for
//        y in [1 + j/128, 1 + (j+1)/128); row 0 = {1/2, 0} for y = 2 exactly; the row is
//        bits 13..20 of y's high word, so y = 2 needs no special case)
#pragma once
#include <cstdint>

namespace plg {

constexpr int kExpBits = 7;
constexpr int kExpN = 1 << kExpBits;  // 128 entries: 2^(j/128)
constexpr int kExpRep = 16;           // lanes per conflict-free group (8-byte slots)
constexpr int kExpRowBytes = kExpRep * 8;
constexpr int kLogBits = 7;
constexpr int kLogRows = 256;
constexpr int kLogRep = 8;            // lanes per conflict-free group (16-byte slots)
constexpr int kLogRowBytes = kLogRep * 16;
constexpr int kExpTableBytes = kExpN * kExpRowBytes;     // 16 KB
constexpr int kLogTableBytes = kLogRows * kLogRowBytes;  // 32 KB
constexpr int kTableBytes = kExpTableBytes + kLogTableBytes;
constexpr int kLogMasterN = (1 << kLogBits) + 1;         // master copy: j = 0..127, then y = 2

// kernels.hpp:17 and kernels.cpp:9
constexpr double kK1 = 79.047;
constexpr double kK2 = 7.4129;
constexpr double kGamma = 0.37457;
constexpr double kGaussianEntropy = 1.4189385332046727418;  // 0.5 * (1 + log(2 pi))
constexpr double kLn2 = 0.69314718055994530942;

constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52: round-to-int in the low word
constexpr double kUScale = 369.32993046757461;  // K = 256 / ln2: callers pass u' = K u
constexpr double kInvUScale = 0.0027076061740622863;  // ln2 / 256

// Coefficients that are not short doubles live in the constant bank (uniform registers
// for the addend slot). Near-minimax degree-4 fits (tools/fit_polys.py, mpmath) whose
// leading coefficient is a short double used as an immediate (kLead*), highest degree
// first:
static __constant__ double kC[12] = {
    -0.00067690154351557160,  // 0  exp(-q/2), q' = u'^2: k = rint(q' * -ln2/1024)
    1477.3197218702985,       // 1                        r' = q' + k * 1024/ln2
    -2.6466431340771855e-08, 1.4662262387638428e-05, -0.005415212348124257,
    //  2-4  exp(-x ln2/128),    |x| <= 0.505:          max rel err 1.6e-16
    -8.20865303897247e-18, 6.718185572625523e-12, -3.6655655969098924e-06,
    //  5-7  exp(-x / (2 K^2)),  |x| <= 1.01 * 512/ln2: max rel err 1.6e-16
    -0.2500025234041795, 0.33333333332155823, -0.4999999999952244,
    //  8-10 log1p(r)/r,         |r| <= 1/257:          max rel err 1.9e-14 (abs of log1p <= 7e-17)
    0.0,
};
constexpr double kLead1 = 3.583033869603014e-11;   // exp1 x^4 (short double)
constexpr double kLead2 = 7.522337778472381e-24;   // exp2 x^4 (short double)
constexpr double kLeadL = 0.20000267028808594;     // log1p x^4 (short double)
// 2^(k/128) scaling is clamped at 2^-100 where the input can leave the normal range: below
// it the term is < 1e-30 absolute (the true value is smaller still).
constexpr int kMinScaledK = -100 * kExpN;

// Fill the shared-memory tables (every thread of the block, then __syncthreads()).
// g_exp: kExpN doubles; g_log: kLogMasterN double2 (host-computed in long double).
// Every thread issues all of its master-copy loads before its first shared store (one L2
// round trip per launch instead of one per entry batch: the fill sits at the start of every
// launch, before any work item, and each pair-list launch pays it).
__device__ __forceinline__ double2 log_master_row(const double2* g_log, int row) {
  double2 v = make_double2(0.0, 0.0);
  if (row == 0) v = g_log[kLogMasterN - 1];
  else if (row >= 128) v = g_log[row - 128];
  return v;
}
__device__ __forceinline__ void load_tables_into(unsigned char* exp_tab, unsigned char* log_tab, const double* g_exp,
                                                 const double2* g_log) {
  double* e = reinterpret_cast<double*>(exp_tab);
  double2* l = reinterpret_cast<double2*>(log_tab);
  constexpr int kNe = kExpN * kExpRep, kNl = kLogRows * kLogRep;  // 2048 each
  constexpr int kPer = 8;
  const int bd = blockDim.x;
  if (bd * kPer >= kNe && bd * kPer >= kNl) {
    double ev[kPer];
    double2 lv[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int i = threadIdx.x + k * bd;
      if (i < kNe) ev[k] = g_exp[i / kExpRep];
      if (i < kNl) lv[k] = log_master_row(g_log, i / kLogRep);
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int i = threadIdx.x + k * bd;
      if (i < kNe) e[i] = ev[k];
      if (i < kNl) l[i] = lv[k];
    }
    return;
  }
  for (int i = threadIdx.x; i < kNe; i += bd) e[i] = g_exp[i / kExpRep];
  for (int i = threadIdx.x; i < kNl; i += bd) l[i] = log_master_row(g_log, i / kLogRep);
}
__device__ __forceinline__ void load_tables(unsigned char* s_tab, const double* g_exp,
                                            const double2* g_log) {
  load_tables_into(s_tab, s_tab + kExpTableBytes, g_exp, g_log);
}

// Per-lane row bases (byte pointers into shared memory).
struct TabPtr {
  const unsigned char* exp;  // + j * kExpRowBytes
  const unsigned char* log;  // + row * kLogRowBytes
};

__device__ __forceinline__ TabPtr table_ptrs(const unsigned char* s_tab, int lane) {
  return {s_tab + (lane & (kExpRep - 1)) * 8, s_tab + kExpTableBytes + (lane & (kLogRep - 1)) * 16};
}

// Alternative table addressing for kernels whose shared-memory base would otherwise cost an
// integer add per lookup: 32-bit shared-window addresses whose table bases are aligned (log
// table 32 KB, exp table 16 KB) so the row offset is OR-ed in by the same LOP3 that masks it.
struct TabAddr {
  uint32_t exp;  // exp table base | lane slot
  uint32_t log;  // log table base | lane slot
};
constexpr int kTableAlignedBytes = kTableBytes + 32768;  // dynamic smem to request (alignment slack)

// Copy the tables into the aligned layout (log at a 32 KB boundary, exp right after it).
__device__ __forceinline__ TabAddr load_tables_aligned(unsigned char* dyn, const double* g_exp, const double2* g_log,
                                                       int lane) {
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(dyn));
  const uint32_t logb = (base + 32767u) & ~32767u;
  const uint32_t expb = logb + kLogTableBytes;  // 32 KB after a 32 KB boundary: 16 KB aligned
  unsigned char* lp = dyn + (logb - base);
  load_tables_into(lp + kLogTableBytes, lp, g_exp, g_log);
  return {expb | static_cast<uint32_t>((lane & (kExpRep - 1)) * 8), logb | static_cast<uint32_t>((lane & (kLogRep - 1)) * 16)};
}

__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ double2 lds_f64x2(uint32_t addr) {
  double2 v;
  asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// 2^(k/128), optionally clamped below at 2^-100. Entry j = k & 127 of the table holds
// 2^(j/128) with j << 13 subtracted from its high word (make_tables), so one integer
// multiply-add of k << 13 into that high word yields 2^(j/128) * 2^(k >> 7) exactly: the
// scaling and the table row come from the same k with no shift/mask pair. The factor is
// normal (>= 2^-866 unclamped for |u| <= sqrt(90000)), so multiplying the polynomial by
// it rounds exactly as scaling the product would.
template <bool kClamp>
__device__ __forceinline__ double exp2_k(const TabPtr& tp, int k) {
  if (kClamp) k = max(k, kMinScaledK);
  const double t = *reinterpret_cast<const double*>(tp.exp + (k & (kExpN - 1)) * kExpRowBytes);
  return __hiloint2double(__double2hiint(t) + k * (1 << (20 - kExpBits)), __double2loint(t));
}

template <bool kClamp>
__device__ __forceinline__ double exp2_k(const TabAddr& tp, int k) {
  if (kClamp) k = max(k, kMinScaledK);
  const double t = lds_f64(tp.exp | (static_cast<uint32_t>(k << 7) & ((kExpN - 1) << 7)));
  return __hiloint2double(__double2hiint(t) + k * (1 << (20 - kExpBits)), __double2loint(t));
}
__device__ __forceinline__ double2 log_row(const TabAddr& tp, unsigned hi) {
  return lds_f64x2(tp.log | ((hi >> (20 - kLogBits - 7)) & ((kLogRows - 1) << 7)));
}
__device__ __forceinline__ double2 log_row(const TabPtr& tp, unsigned hi) {
  const unsigned row = (hi >> (20 - kLogBits)) & (kLogRows - 1);
  return *reinterpret_cast<const double2*>(tp.log + row * kLogRowBytes);
}

// Horner p(x) = 1 + x (c1 + x (c2 + x (c3 + lead x))) with the leading step as
// DMUL-by-immediate + DADD (no contraction).
__device__ __forceinline__ double poly4(double x, double lead, double c3, double c2, double c1) {
  double p = __dadd_rn(__dmul_rn(x, lead), c3);
  p = fma(p, x, c2);
  p = fma(p, x, c1);
  return fma(p, x, 1.0);
}

// Running sums of one residual direction: sum lc = tail + a / K, sum pdf = pdf / K.
struct EdeAcc {
  double tail = 0.0;
  double a = 0.0;
  double pdf = 0.0;
};

// Accumulate one EDE. us = K u (K = 256/ln2). kClampA must be true when |u| can exceed
// ~350 (n > ~1.2e5 samples); |u| <= sqrt(n) for a normalised residual.
template <bool kClampA, typename Tab>
__device__ __forceinline__ void ede_accumulate(double us, EdeAcc& acc, const Tab& tp) {
  // pdf = u exp(-u^2/2) in q' = us^2 units (clamped: q' reaches the subnormal range)
  const double q = us * us;
  const double t2 = fma(q, kC[0], kMagic);
  const int k2 = __double2loint(t2);
  const double r2 = fma(t2 - kMagic, kC[1], q);
  const double e2 = poly4(r2, kLead2, kC[5], kC[6], kC[7]) * exp2_k<true>(tp, k2);
  acc.pdf = fma(us, e2, acc.pdf);
  // exp(-2|u|): k = rint(-|us|), r' = |us| + k, exp(-2|u|) = 2^(k/128) exp(-r' ln2/128)
  const double a = fabs(us);
  const double t1 = kMagic - a;
  const int k1 = __double2loint(t1);
  const double r1 = a + (t1 - kMagic);
  const double v = poly4(r1, kLead1, kC[2], kC[3], kC[4]) * exp2_k<kClampA>(tp, k1);
  // log1p(v) - ln2: y = 1 + v in (1, 2]; r = y c - 1 (one rounding); log y = -log c + log1p(r).
  // The rounding of 1 + v perturbs the result by <= 1.1e-16.
  const double y = 1.0 + v;
  const double2 cl = log_row(tp, static_cast<unsigned>(__double2hiint(y)));
  const double r = fma(y, cl.x, -1.0);
  acc.tail += fma(r, poly4(r, kLeadL, kC[8], kC[9], kC[10]), cl.y);
  acc.a += a;
}

__device__ __forceinline__ double acc_lc(const EdeAcc& acc) { return fma(acc.a, kInvUScale, acc.tail); }
__device__ __forceinline__ double acc_pdf(const EdeAcc& acc) { return acc.pdf * kInvUScale; }

// Entropy from the two sums (kernels.cpp:36-40): H = (kG - (k1 t1) t1) - (k2 t2) t2.
__device__ __forceinline__ double entropy_from_sums(double s_lc, double s_pdf, double inv_n) {
  const double t1 = s_lc * inv_n - kGamma;
  const double t2 = s_pdf * inv_n;
  return (kGaussianEntropy - (kK1 * t1) * t1) - (kK2 * t2) * t2;
}

}  // namespace plg
