// plingam.cpp — host side of the reference API over the B200 engine's C-ABI.
#include "plingam/plingam.hpp"

#include <functional>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>
#include <mutex>

#include "../../../include/plingam_b200.h"

namespace plingam {

const char* to_string(ErrorCode code) {  // error.cpp:5-25
  switch (code) {
    case ErrorCode::NonFinite: return "NonFinite";
    case ErrorCode::ZeroVariance: return "ZeroVariance";
    case ErrorCode::TooFewSamples: return "TooFewSamples";
    case ErrorCode::TooShort: return "TooShort";
    case ErrorCode::LengthMismatch: return "LengthMismatch";
    case ErrorCode::DimensionMismatch: return "DimensionMismatch";
    case ErrorCode::EmptyCandidates: return "EmptyCandidates";
    case ErrorCode::SingularDesign: return "SingularDesign";
    case ErrorCode::InsufficientRows: return "InsufficientRows";
    case ErrorCode::UnstableSystem: return "UnstableSystem";
    case ErrorCode::OutOfRange: return "OutOfRange";
    case ErrorCode::InvalidIndex: return "InvalidIndex";
    case ErrorCode::ParseError: return "ParseError";
    case ErrorCode::IoError: return "IoError";
    case ErrorCode::InvalidFlags: return "InvalidFlags";
    case ErrorCode::EmptyAfterPreprocessing: return "EmptyAfterPreprocessing";
    case ErrorCode::DeviceError: return "DeviceError";
  }
  return "Unknown";
}

std::vector<std::string> default_var_names(std::int64_t dims) {  // types.cpp:9-14
  std::vector<std::string> names;
  names.reserve(static_cast<std::size_t>(dims));
  for (std::int64_t j = 0; j < dims; ++j) names.push_back("x" + std::to_string(j));
  return names;
}

DataMatrix::DataMatrix(std::vector<double> colmajor, std::int64_t m, std::int64_t d,
                       std::vector<std::string> names)
    : values(std::move(colmajor)), rows(m), cols(d), var_names(std::move(names)) {
  if (static_cast<std::int64_t>(values.size()) != m * d)
    throw Error(ErrorCode::DimensionMismatch, "DataMatrix: value count != rows * cols");
  if (var_names.empty()) var_names = default_var_names(d);
}

void validate(const DataMatrix& data) {  // types.cpp:21-47
  if (data.dims() < 1) throw Error(ErrorCode::DimensionMismatch, "validate: need at least 1 variable");
  if (data.samples() < 2) throw Error(ErrorCode::TooFewSamples, "validate: need at least 2 samples");
  if (data.var_names.size() != static_cast<std::size_t>(data.dims()))
    throw Error(ErrorCode::DimensionMismatch, "validate: var_names size mismatch");
  for (std::int64_t j = 0; j < data.dims(); ++j) {
    const auto c = data.col(j);
    for (std::int64_t i = 0; i < data.samples(); ++i)
      if (!std::isfinite(c[static_cast<std::size_t>(i)]))
        throw Error(ErrorCode::NonFinite,
                    "validate: non-finite entry at row " + std::to_string(i) + ", column " +
                        data.var_names[static_cast<std::size_t>(j)],
                    i, j);
    double s = 0.0;
    for (double v : c) s += v;
    const double m = s / static_cast<double>(c.size());
    double q = 0.0;
    for (double v : c) {
      const double dv = v - m;
      q += dv * dv;
    }
    if (q / static_cast<double>(c.size()) == 0.0)
      throw Error(ErrorCode::ZeroVariance,
                  "validate: column " + data.var_names[static_cast<std::size_t>(j)] + " has zero variance", -1, j);
  }
}

bool CausalOrder::is_permutation() const {  // types.cpp:49-60
  const auto d = order.size();
  std::vector<bool> seen(d, false);
  for (int v : order) {
    if (v < 0 || static_cast<std::size_t>(v) >= d || seen[static_cast<std::size_t>(v)]) return false;
    seen[static_cast<std::size_t>(v)] = true;
  }
  return true;
}

std::vector<int> CausalOrder::positions() const {  // types.cpp:62-71
  if (!is_permutation()) throw Error(ErrorCode::InvalidIndex, "positions: order is not a permutation");
  std::vector<int> pos(order.size());
  for (std::size_t p = 0; p < order.size(); ++p) pos[static_cast<std::size_t>(order[p])] = static_cast<int>(p);
  return pos;
}

bool permuted_is_lower_triangular(const WeightedDag& dag) {  // types.cpp:73-88
  const int d = dag.d;
  if (dag.weights.size() != static_cast<std::size_t>(d) * d)
    throw Error(ErrorCode::DimensionMismatch, "permuted_is_lower_triangular: non-square weights");
  if (static_cast<int>(dag.order.order.size()) != d || !dag.order.is_permutation())
    throw Error(ErrorCode::DimensionMismatch,
                "permuted_is_lower_triangular: order is not a permutation of the variables");
  for (std::size_t p = 0; p < dag.order.order.size(); ++p)
    for (std::size_t q = p; q < dag.order.order.size(); ++q)
      if (dag(dag.order.order[p], dag.order.order[q]) != 0.0) return false;
  return true;
}

namespace gpu {

namespace {
// The process-wide context of the reference-shaped API. Calls hold a shared reference for
// their duration, so set_device()/reset() never destroy a context a call is still using
// (the last reference destroys it); plg_ctx serialises concurrent calls on one context.
std::mutex g_mu;
std::shared_ptr<plg_ctx> g_ctx;
int g_device = 0;

std::shared_ptr<plg_ctx> own(plg_ctx* c) { return std::shared_ptr<plg_ctx>(c, [](plg_ctx* p) { plg_ctx_destroy(p); }); }
}  // namespace

void check(int rc, const void* status) {
  if (rc == 0) return;
  const auto* st = static_cast<const plg_status*>(status);
  ErrorCode code = ErrorCode::DeviceError;
  if (st->code >= 1 && st->code <= 16) code = static_cast<ErrorCode>(st->code - 1);
  throw Error(code, st->msg, static_cast<long>(st->row), static_cast<long>(st->col));
}

std::shared_ptr<plg_ctx> context() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_ctx) {
    plg_status st{};
    plg_ctx* c = nullptr;
    check(plg_ctx_create(g_device, &c, &st), &st);
    g_ctx = own(c);
  }
  return g_ctx;
}

void set_device(int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_ctx && device != g_device) g_ctx.reset();
  g_device = device;
}

void reset() {
  std::lock_guard<std::mutex> lk(g_mu);
  g_ctx.reset();
}

std::string nccl_unique_id() {
  std::string id(128, '\0');
  plg_status st{};
  check(plg_nccl_unique_id(id.data(), &st), &st);
  return id;
}

void init_distributed(int device, int rank, int world, const std::string& nccl_uid) {
  if (nccl_uid.size() != 128) throw Error(ErrorCode::OutOfRange, "init_distributed: NCCL id must be 128 bytes");
  std::lock_guard<std::mutex> lk(g_mu);
  g_ctx.reset();
  g_device = device;
  plg_status st{};
  plg_ctx* c = nullptr;
  check(plg_ctx_create_dist(device, rank, world, nccl_uid.data(), &c, &st), &st);
  g_ctx = own(c);
}

void init_peer(int device, int rank, int world, int max_dims,
               const std::function<std::vector<std::string>(const std::string&)>& allgather) {
  plg_status st{};
  plg_ctx* c = nullptr;
  check(plg_ctx_create_p2p(device, rank, world, max_dims, &c, &st), &st);
  auto ctx = own(c);
  std::string mine(64, '\0');
  check(plg_p2p_handle(c, mine.data(), &st), &st);
  const std::vector<std::string> all = allgather(mine);
  if (static_cast<int>(all.size()) != world)
    throw Error(ErrorCode::DimensionMismatch, "init_peer: the exchange returned a handle count != world");
  std::string cat;
  for (const auto& h : all) {
    if (h.size() != 64) throw Error(ErrorCode::OutOfRange, "init_peer: IPC handles are 64 bytes");
    cat += h;
  }
  check(plg_p2p_connect(c, cat.data(), &st), &st);
  std::lock_guard<std::mutex> lk(g_mu);
  g_ctx = ctx;
  g_device = device;
}

}  // namespace gpu

// ordering.cpp:166-168
SearchResult search_causal_order(const DataMatrix& X, std::span<const int> U) {
  SearchResult res;
  res.scores.scores.assign(static_cast<std::size_t>(X.dims()), 0.0);
  std::vector<int32_t> u(U.begin(), U.end());
  plg_status st{};
  gpu::check(plg_search(gpu::context().get(), X.values.data(), X.samples(), static_cast<int32_t>(X.dims()),
                        X.samples(), u.data(), static_cast<int32_t>(u.size()), &res.chosen,
                        res.scores.scores.data(), &st),
             &st);
  return res;
}

// ordering.cpp:170-176
SearchResult search_causal_order_parallel(const DataMatrix& X, std::span<const int> U, int workers) {
  if (workers < 1) throw Error(ErrorCode::OutOfRange, "search_causal_order_parallel: workers must be >= 1");
  return search_causal_order(X, U);
}

// ordering.cpp:178-211
DataMatrix regress_out(const DataMatrix& X, int exog, std::span<const int> remaining) {
  std::vector<int32_t> rem(remaining.begin(), remaining.end());
  std::vector<double> out(static_cast<std::size_t>(X.samples()) * rem.size());
  plg_status st{};
  gpu::check(plg_regress_out(gpu::context().get(), X.values.data(), X.samples(), static_cast<int32_t>(X.dims()),
                             X.samples(), exog, rem.data(), static_cast<int32_t>(rem.size()), out.data(), &st),
             &st);
  std::vector<std::string> names;
  names.reserve(rem.size());
  for (int r : rem) names.push_back(X.var_names[static_cast<std::size_t>(r)]);
  return DataMatrix(std::move(out), X.samples(), static_cast<std::int64_t>(rem.size()), std::move(names));
}

// ordering.cpp:213-244
CausalOrder causal_order(const DataMatrix& X, bool parallel, int workers) {
  (void)parallel;
  if (X.dims() >= 1 && X.samples() >= 2 && X.var_names.size() != static_cast<std::size_t>(X.dims()))
    throw Error(ErrorCode::DimensionMismatch, "validate: var_names size mismatch");
  if (workers < 1) {
    validate(X);
    throw Error(ErrorCode::OutOfRange, "causal_order: workers must be >= 1");
  }
  CausalOrder result;
  result.order.assign(static_cast<std::size_t>(std::max<std::int64_t>(X.dims(), 0)), -1);
  plg_status st{};
  gpu::check(plg_causal_order(gpu::context().get(), X.values.data(), X.samples(), static_cast<int32_t>(X.dims()),
                              std::max<std::int64_t>(X.samples(), 1), result.order.data(), &st),
             &st);
  return result;
}

DirectLingam::DirectLingam(DirectLingamConfig cfg) : cfg_(cfg) {  // direct_lingam.cpp:19-26
  if (cfg_.workers < 1) throw Error(ErrorCode::OutOfRange, "DirectLingam: workers must be >= 1");
  if (cfg_.edge_threshold < 0.0) throw Error(ErrorCode::OutOfRange, "DirectLingam: edge_threshold must be >= 0");
}

WeightedDag DirectLingam::fit(const DataMatrix& X) const {
  FitPhases phases;
  return fit(X, phases);
}

WeightedDag DirectLingam::fit(const DataMatrix& X, FitPhases& phases) const {  // direct_lingam.cpp:33-76
  using Clock = std::chrono::steady_clock;
  const auto t0 = Clock::now();
  CausalOrder order = causal_order(X, cfg_.parallel, cfg_.workers);
  const auto t1 = Clock::now();
  phases.ordering_seconds = std::chrono::duration<double>(t1 - t0).count();
  WeightedDag dag;
  dag.d = static_cast<int>(X.dims());
  dag.weights.assign(static_cast<std::size_t>(dag.d) * dag.d, 0.0);
  dag.intercepts.assign(static_cast<std::size_t>(dag.d), 0.0);
  int32_t used_pinv = 0;
  if (dag.d > 1) {
    plg_status st{};
    gpu::check(plg_fit_weights(gpu::context().get(), X.values.data(), X.samples(), dag.d, X.samples(),
                               order.order.data(), dag.weights.data(), &used_pinv, &st),
               &st);
  }
  dag.used_pinv = used_pinv != 0;
  dag.order = std::move(order);
  const auto t2 = Clock::now();
  phases.weights_seconds = std::chrono::duration<double>(t2 - t1).count();
  phases.total_seconds = std::chrono::duration<double>(t2 - t0).count();
  return dag;
}

EdgeSet to_edges(const WeightedDag& dag, double threshold) {  // direct_lingam.cpp:78-92
  if (threshold < 0.0) throw Error(ErrorCode::OutOfRange, "to_edges: threshold must be >= 0");
  EdgeSet edges;
  for (int i = 0; i < dag.d; ++i)
    for (int j = 0; j < dag.d; ++j) {
      if (i == j) continue;
      if (std::abs(dag(i, j)) > threshold) edges.edges.emplace(j, i);
    }
  return edges;
}

}  // namespace plingam
