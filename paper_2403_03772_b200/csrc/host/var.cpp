// var.cpp — VarLiNGAM front-end.
// estimate_var: proj/src/var_lingam.cpp:7-53 on the B200 (plg_estimate_var: stacked design,
// scaled normal equations by the engine's FP64 Cholesky, residuals on the device).
// estimate_var_qr: the same estimate by one column-pivoted Householder QR on the host, the
// reference's own method, kept as the parity reference of the device path (tests only).
// fit_varlingam restates :55-70 with the causal order and weights from the B200 engine.
#include "plingam/var.hpp"

#include "../../../include/plingam_b200.h"

#include <algorithm>
#include <cmath>
#include <limits>

namespace plingam {

namespace {

// In-place column-pivoted Householder QR of A (m x p, column-major), Eigen-style pivoting
// (largest remaining column norm, LAPACK norm downdates). Returns the numerical rank with
// Eigen's default threshold eps * min(m, p) * |max pivot|.
int colpiv_qr(std::vector<double>& A, int64_t m, int p, std::vector<double>& tau, std::vector<int>& perm) {
  std::vector<double> norms(p), direct(p);
  tau.assign(p, 0.0);
  perm.resize(p);
  for (int j = 0; j < p; ++j) {
    double s = 0.0;
    const double* c = &A[static_cast<size_t>(j) * m];
    for (int64_t i = 0; i < m; ++i) s += c[i] * c[i];
    norms[j] = direct[j] = std::sqrt(s);
    perm[j] = j;
  }
  const int kmax = static_cast<int>(std::min<int64_t>(m, p));
  double maxpiv = 0.0;
  for (int k = 0; k < kmax; ++k) {
    int big = k;
    for (int j = k + 1; j < p; ++j)
      if (norms[j] > norms[big]) big = j;
    if (big != k) {
      std::swap_ranges(A.begin() + static_cast<size_t>(k) * m, A.begin() + static_cast<size_t>(k + 1) * m,
                       A.begin() + static_cast<size_t>(big) * m);
      std::swap(norms[k], norms[big]);
      std::swap(direct[k], direct[big]);
      std::swap(perm[k], perm[big]);
    }
    double* col = &A[static_cast<size_t>(k) * m];
    double tail = 0.0;
    for (int64_t i = k + 1; i < m; ++i) tail += col[i] * col[i];
    const double c0 = col[k];
    double beta = c0, t = 0.0;
    if (tail != 0.0) {
      beta = std::sqrt(c0 * c0 + tail);
      if (c0 >= 0.0) beta = -beta;
      const double denom = c0 - beta;
      for (int64_t i = k + 1; i < m; ++i) col[i] /= denom;
      t = (beta - c0) / beta;
    }
    col[k] = beta;
    tau[k] = t;
    maxpiv = std::max(maxpiv, std::fabs(beta));
    for (int j = k + 1; j < p; ++j) {
      double* cj = &A[static_cast<size_t>(j) * m];
      double s = cj[k];
      for (int64_t i = k + 1; i < m; ++i) s += col[i] * cj[i];
      s *= t;
      cj[k] -= s;
      for (int64_t i = k + 1; i < m; ++i) cj[i] -= s * col[i];
      if (norms[j] != 0.0) {
        double temp = std::fabs(cj[k]) / norms[j];
        temp = std::max(0.0, (1.0 + temp) * (1.0 - temp));
        const double ratio = norms[j] / direct[j];
        if (temp * ratio * ratio <= std::sqrt(std::numeric_limits<double>::epsilon())) {
          double s2 = 0.0;
          for (int64_t i = k + 1; i < m; ++i) s2 += cj[i] * cj[i];
          norms[j] = direct[j] = std::sqrt(s2);
        } else {
          norms[j] *= std::sqrt(temp);
        }
      }
    }
  }
  const double thr = std::numeric_limits<double>::epsilon() * kmax * maxpiv;
  int rank = 0;
  for (int k = 0; k < kmax; ++k)
    if (std::fabs(A[static_cast<size_t>(k) * m + k]) > thr) ++rank;
  return rank;
}

}  // namespace

VarEstimate estimate_var(const DataMatrix& ts, int lag) {
  const int64_t T = ts.samples();
  const int64_t d = ts.dims();
  const int64_t n_rows = T - lag, n_cols = 1 + static_cast<int64_t>(lag) * d;
  std::vector<double> coef(static_cast<size_t>(std::max<int64_t>(n_cols, 1) * std::max<int64_t>(d, 1)));
  std::vector<double> res(static_cast<size_t>(std::max<int64_t>(n_rows, 1) * std::max<int64_t>(d, 1)));
  plg_status st{};
  gpu::check(plg_estimate_var(gpu::context().get(), ts.values.data(), T, static_cast<int32_t>(d), std::max<int64_t>(T, 1),
                              lag, coef.data(), res.data(), &st),
             &st);
  VarEstimate est;
  for (int tau_i = 1; tau_i <= lag; ++tau_i) {  // M_tau(i, j) = coef(1 + (tau-1) d + j, i)
    std::vector<double> M(static_cast<size_t>(d * d));
    for (int64_t i = 0; i < d; ++i)
      for (int64_t j = 0; j < d; ++j)
        M[static_cast<size_t>(j * d + i)] = coef[static_cast<size_t>(i * n_cols + 1 + (tau_i - 1) * d + j)];
    est.m_raw.push_back(std::move(M));
  }
  res.resize(static_cast<size_t>(n_rows * d));
  est.residuals = DataMatrix(std::move(res), n_rows, d, ts.var_names);
  return est;
}

VarEstimate estimate_var_qr(const DataMatrix& ts, int lag) {
  if (lag < 1) throw Error(ErrorCode::OutOfRange, "estimate_var: lag must be >= 1");
  const int64_t T = ts.samples();
  const int64_t d = ts.dims();
  if (d < 1) throw Error(ErrorCode::DimensionMismatch, "estimate_var: need at least 1 variable");
  for (double v : ts.values)
    if (!std::isfinite(v)) throw Error(ErrorCode::NonFinite, "estimate_var: non-finite entries in series");
  const int64_t n_rows = T - lag;
  const int64_t n_cols = 1 + lag * d;
  if (T < lag + 2 * d || n_rows < n_cols)
    throw Error(ErrorCode::InsufficientRows, "estimate_var: series too short for lag " + std::to_string(lag));
  // Z row r (time t = r + lag): [1, x(t-1), ..., x(t-lag)]; Y row r = x(t).
  std::vector<double> Z(static_cast<size_t>(n_rows * n_cols)), Y(static_cast<size_t>(n_rows * d));
  for (int64_t r = 0; r < n_rows; ++r) Z[r] = 1.0;
  for (int tau = 1; tau <= lag; ++tau)
    for (int64_t j = 0; j < d; ++j)
      for (int64_t r = 0; r < n_rows; ++r)
        Z[static_cast<size_t>((1 + (tau - 1) * d + j) * n_rows + r)] = ts(r + lag - tau, j);
  for (int64_t j = 0; j < d; ++j)
    for (int64_t r = 0; r < n_rows; ++r) Y[static_cast<size_t>(j * n_rows + r)] = ts(r + lag, j);
  std::vector<double> QR = Z, tau;
  std::vector<int> perm;
  const int rank = colpiv_qr(QR, n_rows, static_cast<int>(n_cols), tau, perm);
  if (rank < n_cols) throw Error(ErrorCode::SingularDesign, "estimate_var: rank-deficient design matrix");
  // coeffs (n_cols x d) = P R^-1 (Q^T Y)[0:n_cols]
  std::vector<double> coeffs(static_cast<size_t>(n_cols * d));
  std::vector<double> b(static_cast<size_t>(n_rows)), y(static_cast<size_t>(n_cols));
  for (int64_t e = 0; e < d; ++e) {
    std::copy(Y.begin() + e * n_rows, Y.begin() + (e + 1) * n_rows, b.begin());
    for (int64_t k = 0; k < n_cols; ++k) {
      const double* v = &QR[static_cast<size_t>(k * n_rows)];
      double s = b[k];
      for (int64_t i = k + 1; i < n_rows; ++i) s += v[i] * b[i];
      s *= tau[k];
      b[k] -= s;
      for (int64_t i = k + 1; i < n_rows; ++i) b[i] -= s * v[i];
    }
    for (int64_t i = n_cols - 1; i >= 0; --i) {
      double s = b[i];
      for (int64_t j = i + 1; j < n_cols; ++j) s -= QR[static_cast<size_t>(j * n_rows + i)] * y[j];
      y[i] = s / QR[static_cast<size_t>(i * n_rows + i)];
    }
    for (int64_t j = 0; j < n_cols; ++j) coeffs[static_cast<size_t>(e * n_cols + perm[j])] = y[j];
  }
  VarEstimate est;
  for (int tau_i = 1; tau_i <= lag; ++tau_i) {  // M_tau(i, j) = coeffs(1 + (tau-1) d + j, i)
    std::vector<double> M(static_cast<size_t>(d * d));
    for (int64_t i = 0; i < d; ++i)
      for (int64_t j = 0; j < d; ++j)
        M[static_cast<size_t>(j * d + i)] = coeffs[static_cast<size_t>(i * n_cols + 1 + (tau_i - 1) * d + j)];
    est.m_raw.push_back(std::move(M));
  }
  std::vector<double> res(static_cast<size_t>(n_rows * d));
  for (int64_t e = 0; e < d; ++e) {
    double* out = &res[static_cast<size_t>(e * n_rows)];
    for (int64_t r = 0; r < n_rows; ++r) out[r] = Y[static_cast<size_t>(e * n_rows + r)];
    for (int64_t c = 0; c < n_cols; ++c) {
      const double w = coeffs[static_cast<size_t>(e * n_cols + c)];
      const double* zc = &Z[static_cast<size_t>(c * n_rows)];
      for (int64_t r = 0; r < n_rows; ++r) out[r] -= zc[r] * w;
    }
  }
  est.residuals = DataMatrix(std::move(res), n_rows, d, ts.var_names);
  return est;
}

VarModel fit_varlingam(const DataMatrix& ts, int lag, const DirectLingamConfig& cfg) {
  VarEstimate est = estimate_var(ts, lag);
  VarModel model;
  model.lag = lag;
  model.b0 = DirectLingam(cfg).fit(est.residuals);
  model.m_raw = std::move(est.m_raw);
  const int d = model.b0.d;
  // (I - B0) * M_tau on the device (plg_var_lagged_weights)
  const size_t dd = static_cast<size_t>(d) * d;
  std::vector<double> ms(dd * model.m_raw.size()), out(dd * model.m_raw.size());
  for (size_t t = 0; t < model.m_raw.size(); ++t) std::copy(model.m_raw[t].begin(), model.m_raw[t].end(), ms.begin() + t * dd);
  plg_status st{};
  gpu::check(plg_var_lagged_weights(gpu::context().get(), model.b0.weights.data(), ms.data(), d,
                                    static_cast<int32_t>(model.m_raw.size()), out.data(), &st),
             &st);
  for (size_t t = 0; t < model.m_raw.size(); ++t)
    model.b_lagged.emplace_back(out.begin() + t * dd, out.begin() + (t + 1) * dd);
  return model;
}

}  // namespace plingam
