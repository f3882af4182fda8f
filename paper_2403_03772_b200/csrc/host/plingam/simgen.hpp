// simgen.hpp — synthetic LiNGAM inputs (support code for tests and the benchmark).
#pragma once

#include <cstdint>
#include <vector>

#include "plingam/plingam.hpp"

namespace plingam::sim {

enum class NoiseKind { Uniform, Laplace, StudentT3, Gauss };

// Uniform: U(lo, hi) (reference default U(0, 1), simgen.hpp:14-17). Laplace: scale hi.
// StudentT3: hi * t_3. Gauss: N(lo, hi^2) (not identifiable by LiNGAM: the pruning worst case).
struct NoiseSpec {
  NoiseKind kind = NoiseKind::Uniform;
  double lo = 0.0;
  double hi = 1.0;
};

struct Dag {
  int d = 0;
  std::vector<double> weights;  // column-major d x d: weights[v + d*j] = effect of j on v
  std::vector<int> order;       // a causal order of the ground truth
};

Dag gen_two_level_dag(int d, std::uint64_t seed, double edge_prob = 0.5);
Dag gen_sparse_dag(int d, double avg_parents, std::uint64_t seed, double wmin = 0.5, double wmax = 1.5);
// n x d column-major samples.
std::vector<double> sample_lingam(const Dag& dag, std::int64_t n, std::uint64_t seed, const NoiseSpec& noise);

// x(t) = B0 x(t) + sum_tau lagged[tau-1] x(t - tau) + eps(t), burn_in rows discarded
// (simgen.cpp:83-130); the instantaneous system is solved by substitution in B0's causal
// order. lagged[tau]: d x d column-major. Throws UnstableSystem past |x| > 1e9.
// Returns T x d column-major.
std::vector<double> sample_svar(const Dag& b0, const std::vector<std::vector<double>>& lagged, int T,
                                int burn_in, std::uint64_t seed, const NoiseSpec& noise);

// d-vector of U(lo, hi) draws from the seeded generator (e.g. a random lag diagonal).
std::vector<double> uniform_vector(int d, std::uint64_t seed, double lo, double hi);

}  // namespace plingam::sim
