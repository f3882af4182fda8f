// plingam.hpp — the reference's C++ API for the causal-order path, Eigen-free, backed by
// the B200 engine through the C-ABI (include/plingam_b200.h).
//
// Mirrors (paths relative to /root/reference/proj):
//   include/plingam/error.hpp:10-47       ErrorCode, Error
//   include/plingam/types.hpp:17-59       DataMatrix (column-major, contiguous variables),
//                                         validate, CausalOrder, WeightedDag
//   include/plingam/ordering.hpp:13-42    KScores, SearchResult, search_causal_order[_parallel],
//                                         regress_out, causal_order
//   include/plingam/direct_lingam.hpp     DirectLingamConfig (+ gpus), FitPhases, DirectLingam,
//                                         to_edges
// The CPU worker pool is replaced by the GPU engine: `workers`/`parallel` keep their
// argument validation (OutOfRange for workers < 1) and have no other effect, because the
// device result is the same for any worker count (the reference's own bit-identity
// contract, ordering.hpp:29-34). `gpus` selects the number of ranks of a multi-GPU job
// (one process per GPU); it is set up through plingam::gpu::init_distributed.
#pragma once

#include <cstdint>
#include <set>
#include <span>
#include <stdexcept>
#include <memory>
#include <functional>
#include <string>
#include <utility>
#include <vector>

struct plg_ctx;

namespace plingam {

enum class ErrorCode {
  NonFinite,
  ZeroVariance,
  TooFewSamples,
  TooShort,
  LengthMismatch,
  DimensionMismatch,
  EmptyCandidates,
  SingularDesign,
  InsufficientRows,
  UnstableSystem,
  OutOfRange,
  InvalidIndex,
  ParseError,
  IoError,
  InvalidFlags,
  EmptyAfterPreprocessing,
  DeviceError,  // CUDA / NCCL failure: no reference counterpart
};

const char* to_string(ErrorCode code);

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& message, long row = -1, long col = -1)
      : std::runtime_error(message), code_(code), row_(row), col_(col) {}
  ErrorCode code() const noexcept { return code_; }
  long row() const noexcept { return row_; }
  long col() const noexcept { return col_; }

 private:
  ErrorCode code_;
  long row_;
  long col_;
};

// m samples x d variables, column-major: variable j is values[j*m .. j*m+m).
struct DataMatrix {
  std::vector<double> values;
  std::int64_t rows = 0;
  std::int64_t cols = 0;
  std::vector<std::string> var_names;

  DataMatrix() = default;
  DataMatrix(std::vector<double> colmajor, std::int64_t m, std::int64_t d,
             std::vector<std::string> names = {});

  std::int64_t samples() const { return rows; }
  std::int64_t dims() const { return cols; }
  std::span<const double> col(std::int64_t j) const {
    return {values.data() + j * rows, static_cast<std::size_t>(rows)};
  }
  std::span<double> col(std::int64_t j) { return {values.data() + j * rows, static_cast<std::size_t>(rows)}; }
  double& operator()(std::int64_t i, std::int64_t j) { return values[j * rows + i]; }
  double operator()(std::int64_t i, std::int64_t j) const { return values[j * rows + i]; }
};

std::vector<std::string> default_var_names(std::int64_t dims);

// Host restatement of types.cpp:21-47 (the device path validates again on upload).
void validate(const DataMatrix& data);

struct CausalOrder {
  std::vector<int> order;
  bool is_permutation() const;
  std::vector<int> positions() const;
};

struct FitPhases {
  double ordering_seconds = 0.0;
  double weights_seconds = 0.0;
  double total_seconds = 0.0;
};

struct WeightedDag {
  std::vector<double> weights;  // d x d column-major: weights[i + d*j] = effect of j on i
  int d = 0;
  CausalOrder order;
  std::vector<double> intercepts;
  bool used_pinv = false;
  FitPhases phases;  // filled by the fitting calls (the reference returns it separately)
  int dims() const { return d; }
  double operator()(int i, int j) const { return weights[static_cast<std::size_t>(i) + static_cast<std::size_t>(d) * j]; }
};

bool permuted_is_lower_triangular(const WeightedDag& dag);

struct EdgeSet {
  std::set<std::pair<int, int>> edges;
};

struct KScores {
  std::vector<double> scores;
};

struct SearchResult {
  int chosen = -1;
  KScores scores;
};

SearchResult search_causal_order(const DataMatrix& X, std::span<const int> U);
SearchResult search_causal_order_parallel(const DataMatrix& X, std::span<const int> U, int workers);
DataMatrix regress_out(const DataMatrix& X, int exog, std::span<const int> remaining);
CausalOrder causal_order(const DataMatrix& X, bool parallel = false, int workers = 1);

struct DirectLingamConfig {
  bool parallel = false;
  int workers = 1;
  double edge_threshold = 0.05;
};

class DirectLingam {
 public:
  explicit DirectLingam(DirectLingamConfig cfg = {});
  WeightedDag fit(const DataMatrix& X) const;
  WeightedDag fit(const DataMatrix& X, FitPhases& phases) const;
  const DirectLingamConfig& config() const { return cfg_; }

 private:
  DirectLingamConfig cfg_;
};

EdgeSet to_edges(const WeightedDag& dag, double threshold);

namespace gpu {

// The engine the API above runs on: device `device` (default: the current CUDA device,
// 0 if none set), single rank unless init_distributed was called.
std::shared_ptr<plg_ctx> context();
// One process per GPU: every rank calls this with the same 128-byte NCCL unique id
// (nccl_unique_id() on rank 0, broadcast by the caller). Replaces context().
void init_distributed(int device, int rank, int world, const std::string& nccl_uid);
// Multi-GPU through peer memory (plg_ctx_create_p2p): allgather(this rank's 64-byte IPC
// handle) must return every rank's handle in rank order (any host channel).
void init_peer(int device, int rank, int world, int max_dims,
               const std::function<std::vector<std::string>(const std::string&)>& allgather);
std::string nccl_unique_id();
void set_device(int device);
void reset();

// Throw plingam::Error for a failed C-ABI status.
void check(int rc, const void* status);

}  // namespace gpu

}  // namespace plingam
