// plg_math.cuh — FP64 element math of the entropy approximation, sm_100a.
//
// One "EDE" (element-direction evaluation) is one sample u of one residual entropy
// (reference proj/src/kernels.cpp:16-34):
//     lc  = |u| + (log1p(exp(-2|u|)) - ln2)      (log cosh u)
//     pdf = u * exp(-u^2 / 2)
// libdevice exp + log1p + exp cost ~70 FP64-pipe instructions per EDE. Here both
// exponentials use a 128-entry 2^(j/128) table (|reduced arg| <= ln2/256, degree-5
// Taylor) and log1p uses a 129-entry reciprocal/log table (|r| <= 1/257, degree-5
// Taylor), which brings an EDE to ~32 FP64 instructions. Absolute error per element
// is <= ~2e-15 in lc and pdf (tests/test_gpu_math.py checks this against libdevice);
// the causal order needs ~1e-9.
//
// The tables live in shared memory, replicated per lane group so that random
// per-lane indices never bank-conflict: the exp table is interleaved 16-way
// (one 8-byte slot per lane of a half-warp), the log table 8-way (16-byte slots,
// one per lane of a quarter-warp).
#pragma once
#include <cstdint>

namespace plg {

constexpr int kExpBits = 7;
constexpr int kExpN = 1 << kExpBits;       // 128 entries: 2^(j/128)
constexpr int kExpRep = 16;                // lanes per conflict-free group (8-byte slots)
constexpr int kLogBits = 7;
constexpr int kLogN = (1 << kLogBits) + 1; // 129 entries: y in [1 + j/128, 1 + (j+1)/128), j=128 <-> y=2
constexpr int kLogRep = 8;                 // lanes per conflict-free group (16-byte slots)
constexpr int kTableBytes = kExpN * kExpRep * 8 + kLogN * kLogRep * 16;

// kernels.hpp:17 and kernels.cpp:9
constexpr double kK1 = 79.047;
constexpr double kK2 = 7.4129;
constexpr double kGamma = 0.37457;
constexpr double kGaussianEntropy = 1.4189385332046727418;  // 0.5 * (1 + log(2 pi))
constexpr double kLn2 = 0.69314718055994530942;

constexpr double kMagic = 6755399441055744.0;   // 1.5 * 2^52: round-to-int in the low word
constexpr double kExpA = -256.0 / kLn2;         // exp(-2a):  k = rint(-2a * 128 / ln2)
constexpr double kExpARed = kLn2 / 256.0;       //            r' = a + k ln2/256, exp(-2a) = 2^(k/128) e^(-2 r')
constexpr double kExpQ = -64.0 / kLn2;          // exp(-q/2): k = rint(-q/2 * 128 / ln2)
constexpr double kExpQRed = kLn2 / 64.0;        //            r' = q + k ln2/64,  exp(-q/2) = 2^(k/128) e^(-r'/2)

// Clamps (applied to the high word, i.e. to within one ulp of the bound): beyond them
// the term is below 1e-34 absolute and the table scaling would leave the normal range.
constexpr int kHiA40 = 0x40440000;    // high word of 40.0
constexpr int kHiQ1400 = 0x4095E000;  // high word of 1400.0

struct Tables {
  const double* exp_tab;   // [kExpN][kExpRep]
  const double2* log_tab;  // [kLogN][kLogRep]: {c_j, -log(c_j) - ln2}
};

// Fill the shared-memory tables (called by every thread of the block, then sync).
// Host-precomputed master copies live in global memory (computed in long double,
// see engine.cu make_tables()).
__device__ __forceinline__ void load_tables(double* s_exp, double2* s_log, const double* g_exp,
                                            const double2* g_log) {
  for (int i = threadIdx.x; i < kExpN * kExpRep; i += blockDim.x) s_exp[i] = g_exp[i / kExpRep];
  for (int i = threadIdx.x; i < kLogN * kLogRep; i += blockDim.x) s_log[i] = g_log[i / kLogRep];
}

__device__ __forceinline__ double scale_pow2(double v, int k) {
  // v * 2^(k >> 7): add to the exponent field; arguments are clamped so the result
  // stays normal.
  const int hi = __double2hiint(v) + ((k >> kExpBits) << 20);
  return __hiloint2double(hi, __double2loint(v));
}

// exp(-2a) for a >= 0 (a already clamped to <= 40).
__device__ __forceinline__ double exp_m2a(double a, const double* exp_row) {
  const double t = fma(a, kExpA, kMagic);
  const int k = __double2loint(t);
  const double kd = t - kMagic;
  const double r = fma(kd, kExpARed, a);  // exp(-2a) = 2^(k/128) * exp(-2r)
  // exp(-2r) = sum (-2r)^i / i!, |2r| <= ln2/128
  double p = fma(r, -4.0 / 15.0, 2.0 / 3.0);  // (-2)^5/120, (-2)^4/24
  p = fma(p, r, -4.0 / 3.0);                  // (-2)^3/6
  p = fma(p, r, 2.0);                         // (-2)^2/2
  p = fma(p, r, -2.0);
  p = fma(p, r, 1.0);
  const double v = p * exp_row[(k & (kExpN - 1)) * kExpRep];
  return scale_pow2(v, k);
}

// exp(-q/2) for q >= 0 (q already clamped to <= 1400).
__device__ __forceinline__ double exp_mhalf(double q, const double* exp_row) {
  const double t = fma(q, kExpQ, kMagic);
  const int k = __double2loint(t);
  const double kd = t - kMagic;
  const double r = fma(kd, kExpQRed, q);  // exp(-q/2) = 2^(k/128) * exp(-r/2)
  // exp(-r/2) = sum (-r/2)^i / i!, |r/2| <= ln2/256
  double p = fma(r, -1.0 / 3840.0, 1.0 / 384.0);  // (-1/2)^5/120, (-1/2)^4/24
  p = fma(p, r, -1.0 / 48.0);                     // (-1/2)^3/6
  p = fma(p, r, 1.0 / 8.0);                       // (-1/2)^2/2
  p = fma(p, r, -0.5);
  p = fma(p, r, 1.0);
  const double v = p * exp_row[(k & (kExpN - 1)) * kExpRep];
  return scale_pow2(v, k);
}

// |u| + log1p(v) - ln2 for v in (0, 1]: y = 1 + v in (1, 2]; j = top 7 mantissa bits
// (j = 128 exactly at y = 2); r = y c_j - 1 (one rounding, FMA); log y = -log c_j + log1p(r).
// The rounding of 1 + v perturbs the result by <= 1.1e-16 absolute.
__device__ __forceinline__ double logcosh_tail(double a, double v, const double2* log_row) {
  const double y = 1.0 + v;
  const int j = (__double2hiint(y) - 0x3FF00000) >> (20 - kLogBits);
  const double2 cl = log_row[j * kLogRep];
  const double r = fma(y, cl.x, -1.0);
  // log1p(r) = r (1 - r/2 + r^2/3 - r^3/4 + r^4/5), |r| <= 1/257
  double p = fma(r, 0.2, -0.25);
  p = fma(p, r, 1.0 / 3.0);
  p = fma(p, r, -0.5);
  p = fma(p, r, 1.0);
  return fma(r, p, a + cl.y);
}

// Accumulate one EDE of sample u into (s_lc, s_pdf).
__device__ __forceinline__ void ede_accumulate(double u, double& s_lc, double& s_pdf,
                                               const double* exp_row, const double2* log_row) {
  const double a = fabs(u);
  const double ac = __hiloint2double(min(__double2hiint(a), kHiA40), __double2loint(a));
  const double v = exp_m2a(ac, exp_row);
  s_lc += logcosh_tail(a, v, log_row);
  const double q = u * u;
  const double qc = __hiloint2double(min(__double2hiint(q), kHiQ1400), __double2loint(q));
  const double e = exp_mhalf(qc, exp_row);
  s_pdf = fma(u, e, s_pdf);
}

// Entropy from the two sums (kernels.cpp:36-40): H = (kG - (k1 t1) t1) - (k2 t2) t2.
__device__ __forceinline__ double entropy_from_sums(double s_lc, double s_pdf, double inv_n) {
  const double t1 = s_lc * inv_n - kGamma;
  const double t2 = s_pdf * inv_n;
  return (kGaussianEntropy - (kK1 * t1) * t1) - (kK2 * t2) * t2;
}

}  // namespace plg
