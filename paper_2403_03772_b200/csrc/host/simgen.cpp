// simgen.cpp — synthetic inputs for the benchmark configurations (BASELINE.json configs).
//
// Support code, not the hot path. The generators follow the reference's semantics
// (proj/include/plingam/rng.hpp:14-43: mt19937_64, 53-bit uniforms, Box-Muller,
// Fisher-Yates; proj/src/simgen.cpp:30-81: two-level DAG, causal-order sampling) and add
// the shapes the configs name that the reference has no generator for (sparse
// Erdos-Renyi DAGs, Laplace and heavy-tailed noise).
#include "plingam/simgen.hpp"

#include <cmath>
#include <numbers>
#include <random>

namespace plingam::sim {

namespace {

class Rng {  // rng.hpp:14-43
 public:
  explicit Rng(std::uint64_t seed) : gen_(seed) {}
  double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double gauss() {
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::numbers::pi * u2);
  }
  template <typename T>
  void shuffle(std::vector<T>& v) {
    for (std::size_t i = v.size(); i > 1; --i) {
      auto j = static_cast<std::size_t>(uniform() * static_cast<double>(i));
      std::swap(v[i - 1], v[j]);
    }
  }

 private:
  std::mt19937_64 gen_;
};

double draw_noise(Rng& rng, const NoiseSpec& noise) {
  switch (noise.kind) {
    case NoiseKind::Uniform:
      return rng.uniform(noise.lo, noise.hi);
    case NoiseKind::Laplace: {  // inverse CDF, scale b = noise.hi
      const double p = rng.uniform() - 0.5;
      const double a = 1.0 - 2.0 * std::fabs(p);
      return -noise.hi * (p < 0 ? -1.0 : 1.0) * std::log(a > 0 ? a : 0x1.0p-53);
    }
    case NoiseKind::StudentT3: {  // heavy-tailed: t with 3 degrees of freedom
      const double z = rng.gauss();
      double chi = 0.0;
      for (int k = 0; k < 3; ++k) {
        const double g = rng.gauss();
        chi += g * g;
      }
      return noise.hi * z / std::sqrt(chi / 3.0);
    }
    case NoiseKind::Gauss:
      return noise.lo + noise.hi * rng.gauss();
  }
  return 0.0;
}

}  // namespace

Dag gen_two_level_dag(int d, std::uint64_t seed, double edge_prob) {  // simgen.cpp:30-57
  if (d < 2) throw Error(ErrorCode::OutOfRange, "simgen: dims must be >= 2");
  if (!(edge_prob > 0.0) || edge_prob > 1.0) throw Error(ErrorCode::OutOfRange, "simgen: edge_prob must be in (0, 1]");
  const int n0 = (d + 1) / 2;
  Rng rng(seed);
  Dag dag;
  dag.d = d;
  dag.weights.assign(static_cast<std::size_t>(d) * d, 0.0);
  dag.order.resize(static_cast<std::size_t>(d));
  for (int v = 0; v < d; ++v) dag.order[static_cast<std::size_t>(v)] = v;
  rng.shuffle(dag.order);
  for (int u = 0; u < n0; ++u)
    for (int v = n0; v < d; ++v)
      if (rng.uniform() < edge_prob) {
        const double w = rng.gauss();
        dag.weights[static_cast<std::size_t>(dag.order[v]) + static_cast<std::size_t>(d) * dag.order[u]] = w;
      }
  return dag;
}

Dag gen_sparse_dag(int d, double avg_parents, std::uint64_t seed, double wmin, double wmax) {
  if (d < 2) throw Error(ErrorCode::OutOfRange, "simgen: dims must be >= 2");
  Rng rng(seed);
  Dag dag;
  dag.d = d;
  dag.weights.assign(static_cast<std::size_t>(d) * d, 0.0);
  dag.order.resize(static_cast<std::size_t>(d));
  for (int v = 0; v < d; ++v) dag.order[static_cast<std::size_t>(v)] = v;
  rng.shuffle(dag.order);
  // Erdos-Renyi over the order: each earlier node is a parent with probability
  // p = 2 * avg_parents / (d - 1), so the expected in-degree averages avg_parents.
  const double p = std::min(1.0, 2.0 * avg_parents / static_cast<double>(d - 1));
  for (int b = 1; b < d; ++b)
    for (int a = 0; a < b; ++a)
      if (rng.uniform() < p) {
        const double mag = rng.uniform(wmin, wmax);
        const double w = rng.uniform() < 0.5 ? -mag : mag;
        dag.weights[static_cast<std::size_t>(dag.order[b]) + static_cast<std::size_t>(d) * dag.order[a]] = w;
      }
  return dag;
}

std::vector<double> sample_lingam(const Dag& dag, std::int64_t n, std::uint64_t seed, const NoiseSpec& noise) {
  // simgen.cpp:59-81: per row, one noise draw per variable in index order, then
  // x_v = sum_j w(v, j) x_j + eps_v in causal order. Sparse parents.
  const int d = dag.d;
  std::vector<std::vector<std::pair<int, double>>> parents(static_cast<std::size_t>(d));
  for (int v = 0; v < d; ++v)
    for (int j = 0; j < d; ++j) {
      const double w = dag.weights[static_cast<std::size_t>(v) + static_cast<std::size_t>(d) * j];
      if (w != 0.0) parents[static_cast<std::size_t>(v)].emplace_back(j, w);
    }
  Rng rng(seed);
  std::vector<double> X(static_cast<std::size_t>(n) * d);
  std::vector<double> eps(static_cast<std::size_t>(d)), x(static_cast<std::size_t>(d));
  for (std::int64_t r = 0; r < n; ++r) {
    for (int j = 0; j < d; ++j) eps[static_cast<std::size_t>(j)] = draw_noise(rng, noise);
    for (int v : dag.order) {
      double s = 0.0;
      for (const auto& [j, w] : parents[static_cast<std::size_t>(v)]) s += w * x[static_cast<std::size_t>(j)];
      x[static_cast<std::size_t>(v)] = s + eps[static_cast<std::size_t>(v)];
    }
    for (int j = 0; j < d; ++j) X[static_cast<std::size_t>(r) + static_cast<std::size_t>(n) * j] = x[static_cast<std::size_t>(j)];
  }
  return X;
}

std::vector<double> sample_svar(const Dag& b0, const std::vector<std::vector<double>>& lagged, int T,
                                int burn_in, std::uint64_t seed, const NoiseSpec& noise) {
  const int d = b0.d;
  for (const auto& m : lagged)
    if (m.size() != static_cast<std::size_t>(d) * d)
      throw Error(ErrorCode::DimensionMismatch, "sample_svar: lagged matrix shape mismatch");
  if (T < 1 || burn_in < 0) throw Error(ErrorCode::OutOfRange, "sample_svar: need T >= 1 and burn_in >= 0");
  std::vector<std::vector<std::pair<int, double>>> parents(static_cast<std::size_t>(d));
  for (int v = 0; v < d; ++v)
    for (int j = 0; j < d; ++j) {
      const double w = b0.weights[static_cast<std::size_t>(v) + static_cast<std::size_t>(d) * j];
      if (w != 0.0) parents[static_cast<std::size_t>(v)].emplace_back(j, w);
    }
  const int k = static_cast<int>(lagged.size());
  Rng rng(seed);
  std::vector<std::vector<double>> history(static_cast<std::size_t>(k), std::vector<double>(d, 0.0));
  std::vector<double> out(static_cast<std::size_t>(T) * d), rhs(d), x(d);
  for (int t = 0; t < burn_in + T; ++t) {
    for (int j = 0; j < d; ++j) rhs[j] = draw_noise(rng, noise);
    for (int tau = 0; tau < k; ++tau) {
      const auto& M = lagged[static_cast<std::size_t>(tau)];
      const auto& h = history[static_cast<std::size_t>(tau)];
      for (int j = 0; j < d; ++j) {
        const double hj = h[j];
        if (hj == 0.0) continue;
        for (int i = 0; i < d; ++i) rhs[i] += M[static_cast<std::size_t>(j) * d + i] * hj;
      }
    }
    for (int v : b0.order) {  // (I - B0) x = rhs by substitution in causal order
      double s = rhs[v];
      for (const auto& [j, w] : parents[static_cast<std::size_t>(v)]) s += w * x[j];
      x[v] = s;
    }
    for (int j = 0; j < d; ++j)
      if (!std::isfinite(x[j]) || std::fabs(x[j]) > 1e9)
        throw Error(ErrorCode::UnstableSystem, "sample_svar: series exceeded overflow guard");
    for (int tau = k - 1; tau > 0; --tau) history[static_cast<std::size_t>(tau)] = history[static_cast<std::size_t>(tau - 1)];
    if (k > 0) history[0] = x;
    if (t >= burn_in)
      for (int j = 0; j < d; ++j) out[static_cast<std::size_t>(t - burn_in) + static_cast<std::size_t>(T) * j] = x[j];
  }
  return out;
}

std::vector<double> uniform_vector(int d, std::uint64_t seed, double lo, double hi) {
  Rng rng(seed);
  std::vector<double> v(static_cast<std::size_t>(d));
  for (auto& x : v) x = rng.uniform(lo, hi);
  return v;
}

}  // namespace plingam::sim
