// var.hpp — VarLiNGAM front-end: the VAR(k) estimate whose residuals
// feed the causal-order engine, and the lag transform. Restates (paths relative to
// /root/reference/proj) include/plingam/var_lingam.hpp:13-39 and src/var_lingam.cpp:7-70.
#pragma once

#include <vector>

#include "plingam/plingam.hpp"

namespace plingam {

struct VarEstimate {
  std::vector<std::vector<double>> m_raw;  // M_1..M_k, each d x d column-major
  DataMatrix residuals;                    // (T - k) x d
};

// Least-squares VAR(k) with intercept (estimated, then discarded) of the stacked design
// [1, x(t-1), ..., x(t-k)] (var_lingam.cpp:7-53), on the B200 (plg_estimate_var).
// `ts` rows are time points. Throws OutOfRange (lag < 1), DimensionMismatch, NonFinite,
// InsufficientRows and SingularDesign.
VarEstimate estimate_var(const DataMatrix& ts, int lag);
// The same estimate by the reference's method (column-pivoted Householder QR on the host):
// the parity reference of estimate_var's device path, used by the tests.
VarEstimate estimate_var_qr(const DataMatrix& ts, int lag);

struct VarModel {
  WeightedDag b0;
  std::vector<std::vector<double>> b_lagged;  // (I - B0) M_tau, d x d column-major
  std::vector<std::vector<double>> m_raw;
  int lag = 0;
};

// VAR estimate, DirectLiNGAM (GPU causal order + weights) on the residuals, then
// b_lagged[tau] = (I - B0) * m_raw[tau] (var_lingam.cpp:55-70).
VarModel fit_varlingam(const DataMatrix& ts, int lag, const DirectLingamConfig& cfg = {});

}  // namespace plingam
