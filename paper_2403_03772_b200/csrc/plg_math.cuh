// plg_math.cuh — FP64 element math of the entropy approximation, sm_100a.
//
// One "EDE" (element-direction evaluation) is one sample u of one residual entropy
// (reference proj/src/kernels.cpp:16-34):
//     lc  = |u| + (log1p(exp(-2|u|)) - ln2)      (log cosh u)
//     pdf = u * exp(-u^2 / 2)
// libdevice exp + log1p + exp cost ~70 FP64-pipe instructions per EDE. Here both
// exponentials use a 128-entry 2^(j/128) table (|reduced arg| <= ln2/256) and log1p a
// 128-entry reciprocal/log table (|r| <= 1/257), each finished by a degree-4 near-minimax
// polynomial (tools/fit_polys.py): 29 FP64 instructions per EDE plus ~20 integer/LDS ones
// (index and exponent arithmetic, table reads), checked in SASS. Absolute error per
// element is a few ulp of lc and pdf (tests/test_gpu_parity.py checks against libdevice
// and numpy); the causal order needs ~1e-9.
//
// Throughput is bound by register-file reads rather than by the FP64 pipe itself: a DFMA
// reading 3 distinct register pairs takes 3 issue cycles instead of 2, and integer
// instructions share the read ports (measured, tools/probe/fp64_mix.cu; model and SASS
// census in tools/rf_model.py, which predicts the measured 69% FP64-pipe utilisation).
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

// Coefficients that are not short doubles live in the constant bank: ptxas loads them
// once (uniform registers for DFMA's addend slot) instead of re-materialising register
// pairs every iteration (measured: -20 issue slots per 8 EDE in the pair kernel's loop).
static __constant__ double kC[16] = {
    -256.0 / kLn2,  // 0  exp(-2a):  k = rint(-2a * 128 / ln2)
    kLn2 / 256.0,   // 1            r = a + k ln2/256, exp(-2a) = 2^(k/128) e^(-2r)
    -64.0 / kLn2,   // 2  exp(-q/2): k = rint(-q/2 * 128 / ln2)
    kLn2 / 64.0,    // 3            r = q + k ln2/64,  exp(-q/2) = 2^(k/128) e^(-r/2)
    // near-minimax degree-4 fits (tools/fit_polys.py, mpmath), highest degree first:
    0.6666668744024424, -1.3333339565406885, 1.999999999999903, -1.9999999999997087,
    //   4-7  exp(-2r),   |r| <= 1.01 ln2/512: max rel err 8.0e-17
    0.0026041674781345408, -0.02083334307094826, 0.12499999999999394, -0.49999999999992717,
    //   8-11 exp(-r/2),  |r| <= 1.01 ln2/128: max rel err 8.0e-17
    0.20000270365230982, -0.25000315425970154, 0.3333333333230998, -0.4999999999880609,
    //  12-15 log1p(r)/r, |r| <= 1/257: max rel err 9.3e-15 (abs err of log1p <= 3.6e-17)
};
// 2^(k/128) scaling is clamped at 2^-100: below it the term is < 1e-30 absolute (the true
// value is smaller still) and the exponent field stays normal for any finite input.
constexpr int kMinScaledK = -100 * kExpN;

// Fill the shared-memory tables (every thread of the block, then __syncthreads()).
// g_exp: kExpN doubles; g_log: kLogMasterN double2 (host-computed in long double).
__device__ __forceinline__ void load_tables(unsigned char* s_tab, const double* g_exp,
                                            const double2* g_log) {
  double* e = reinterpret_cast<double*>(s_tab);
  for (int i = threadIdx.x; i < kExpN * kExpRep; i += blockDim.x) e[i] = g_exp[i / kExpRep];
  double2* l = reinterpret_cast<double2*>(s_tab + kExpTableBytes);
  for (int i = threadIdx.x; i < kLogRows * kLogRep; i += blockDim.x) {
    const int row = i / kLogRep;
    double2 v = make_double2(0.0, 0.0);
    if (row == 0) v = g_log[kLogMasterN - 1];
    else if (row >= 128) v = g_log[row - 128];
    l[i] = v;
  }
}

// Per-lane row bases (byte pointers into shared memory).
struct TabPtr {
  const unsigned char* exp;  // + j * kExpRowBytes
  const unsigned char* log;  // + row * kLogRowBytes
};

__device__ __forceinline__ TabPtr table_ptrs(const unsigned char* s_tab, int lane) {
  return {s_tab + (lane & (kExpRep - 1)) * 8, s_tab + kExpTableBytes + (lane & (kLogRep - 1)) * 16};
}

// v * 2^(k >> 7) with k clamped: add (k & ~127) << 13 to the high word (one IMAD).
__device__ __forceinline__ double scale_pow2(double v, int k) {
  const int kh = max(k & ~(kExpN - 1), kMinScaledK);
  return __hiloint2double(__double2hiint(v) + kh * (1 << (20 - kExpBits)), __double2loint(v));
}

__device__ __forceinline__ double exp_row(const TabPtr& tp, int k) {
  return *reinterpret_cast<const double*>(tp.exp + (k & (kExpN - 1)) * kExpRowBytes);
}

// exp(-2a) for a >= 0.
__device__ __forceinline__ double exp_m2a(double a, const TabPtr& tp) {
  const double t = fma(a, kC[0], kMagic);
  const int k = __double2loint(t);
  const double kd = t - kMagic;
  const double r = fma(kd, kC[1], a);  // exp(-2a) = 2^(k/128) * exp(-2r), |2r| <= ln2/128
  double p = fma(r, kC[4], kC[5]);
  p = fma(p, r, kC[6]);
  p = fma(p, r, kC[7]);
  p = fma(p, r, 1.0);
  return scale_pow2(p * exp_row(tp, k), k);
}

// exp(-q/2) for q >= 0.
__device__ __forceinline__ double exp_mhalf(double q, const TabPtr& tp) {
  const double t = fma(q, kC[2], kMagic);
  const int k = __double2loint(t);
  const double kd = t - kMagic;
  const double r = fma(kd, kC[3], q);  // exp(-q/2) = 2^(k/128) * exp(-r/2), |r/2| <= ln2/256
  double p = fma(r, kC[8], kC[9]);
  p = fma(p, r, kC[10]);
  p = fma(p, r, kC[11]);
  p = fma(p, r, 1.0);
  return scale_pow2(p * exp_row(tp, k), k);
}

// a + log1p(v) - ln2 for v in (0, 1]: y = 1 + v in (1, 2]; r = y c - 1 (one rounding);
// log y = -log c + log1p(r). The rounding of 1 + v perturbs the result by <= 1.1e-16.
__device__ __forceinline__ double logcosh_tail(double a, double v, const TabPtr& tp) {
  const double y = 1.0 + v;
  const unsigned row = (static_cast<unsigned>(__double2hiint(y)) >> (20 - kLogBits)) & (kLogRows - 1);
  const double2 cl = *reinterpret_cast<const double2*>(tp.log + row * kLogRowBytes);
  const double r = fma(y, cl.x, -1.0);
  double p = fma(r, kC[12], kC[13]);  // log1p(r) = r p(r)
  p = fma(p, r, kC[14]);
  p = fma(p, r, kC[15]);
  p = fma(p, r, 1.0);
  return fma(r, p, a + cl.y);
}

__device__ __forceinline__ double abs_int(double u) {  // |u| on the integer pipe
  return __hiloint2double(__double2hiint(u) & 0x7fffffff, __double2loint(u));
}

// Accumulate one EDE of sample u into (s_lc, s_pdf).
__device__ __forceinline__ void ede_accumulate(double u, double& s_lc, double& s_pdf, const TabPtr& tp) {
  s_pdf = fma(u, exp_mhalf(u * u, tp), s_pdf);
  const double a = abs_int(u);
  s_lc += logcosh_tail(a, exp_m2a(a, tp), tp);
}

// Entropy from the two sums (kernels.cpp:36-40): H = (kG - (k1 t1) t1) - (k2 t2) t2.
__device__ __forceinline__ double entropy_from_sums(double s_lc, double s_pdf, double inv_n) {
  const double t1 = s_lc * inv_n - kGamma;
  const double t2 = s_pdf * inv_n;
  return (kGaussianEntropy - (kK1 * t1) * t1) - (kK2 * t2) * t2;
}

}  // namespace plg
