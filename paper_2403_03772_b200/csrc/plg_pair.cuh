// plg_pair.cuh — per-pair residual scales from the maintained Gram (shared by every pair
// kernel so that E(i|j) has the same bits whichever kernel evaluates the pair).
#pragma once
#include <cstdint>

#include "plg_math.cuh"

namespace plg {

// Scales of both directions of pair (i, j): u'_1 = x s1 - y bs1 is the K-scaled residual of
// i on j (slope b1 = C_ij / C_jj, ordering.cpp:89), u'_2 = y s2 - x bs2 that of j on i
// (b2 = C_ij / C_ii, ordering.cpp:90); x = w_i, y = w_j. Symmetric in (i, j) given a
// bit-symmetric C. Returns false (scales zero) for an exactly collinear pair, whose residual
// is identically zero (entropy_of_normalized throws, kernels.cpp:136-139).
// Slopes and residual variances of a pair from its Gram entries (explicitly rounded, so every
// kernel that tests or uses them gets the same bits).
__device__ __forceinline__ void pair_vars(double cii, double cjj, double cij, double& b1, double& v1,
                                          double& b2, double& v2) {
  b1 = __ddiv_rn(cij, cjj);
  v1 = __dsub_rn(cii, __dmul_rn(cij, b1));
  b2 = __ddiv_rn(cij, cii);
  v2 = __dsub_rn(cjj, __dmul_rn(cij, b2));
}
__device__ __forceinline__ bool pair_collinear(double v1, double v2) { return !(v1 > 0.0) || !(v2 > 0.0); }

__device__ __forceinline__ bool pair_scales(const double* C, int64_t ldc, int ci, int cj, double& s1,
                                            double& bs1, double& s2, double& bs2) {
  const double cii = C[static_cast<int64_t>(ci) * ldc + ci];
  const double cjj = C[static_cast<int64_t>(cj) * ldc + cj];
  const double cij = C[static_cast<int64_t>(ci) * ldc + cj];
  double b1, v1, b2, v2;
  pair_vars(cii, cjj, cij, b1, v1, b2, v2);
  if (pair_collinear(v1, v2)) {
    s1 = bs1 = s2 = bs2 = 0.0;
    return false;
  }
  s1 = kUScale / sqrt(v1);
  bs1 = b1 * s1;
  s2 = kUScale / sqrt(v2);
  bs2 = b2 * s2;
  return true;
}

}  // namespace plg
