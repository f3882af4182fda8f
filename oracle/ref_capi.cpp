// ref_capi.cpp — TEST INFRASTRUCTURE ONLY: a C entry point to the reference's own
// causal-order code (proj/src/{kernels,ordering,types,error}.cpp compiled unmodified against
// oracle/eigen_shim by oracle/Makefile.ref into oracle/_ref/libplingam_ref.so), so that the
// oracle restatement, the bench's reference arm and the GPU results can be checked against
// the reference implementation itself.
#include <cstdint>
#include <cstring>
#include <span>
#include <vector>

#include "plingam/ordering.hpp"

namespace {
plingam::DataMatrix to_data(const double* X, int64_t n, int32_t d) {
  Eigen::MatrixXd m(n, d);
  std::memcpy(m.data(), X, sizeof(double) * static_cast<std::size_t>(n) * static_cast<std::size_t>(d));
  return plingam::DataMatrix(std::move(m));
}
int fail(const plingam::Error& e, int32_t* code, int64_t* row, int64_t* col) {
  *code = 1 + static_cast<int32_t>(e.code());
  *row = e.row();
  *col = e.col();
  return *code;
}
}  // namespace

extern "C" {

// plingam::causal_order(X, parallel, workers) (ordering.hpp:42); X column-major n x d.
int ref_causal_order(const double* X, int64_t n, int32_t d, int32_t parallel, int32_t workers, int32_t* order_out,
                     int32_t* code, int64_t* row, int64_t* col) {
  *code = 0;
  try {
    const plingam::CausalOrder o = plingam::causal_order(to_data(X, n, d), parallel != 0, workers);
    for (std::size_t i = 0; i < o.order.size(); ++i) order_out[i] = o.order[i];
    return 0;
  } catch (const plingam::Error& e) {
    return fail(e, code, row, col);
  }
}

// plingam::search_causal_order[_parallel](X, U) (ordering.hpp:27-34): chosen and the d scores.
int ref_search(const double* X, int64_t n, int32_t d, const int32_t* U, int32_t u, int32_t workers,
               int32_t* chosen_out, double* scores_out, int32_t* code, int64_t* row, int64_t* col) {
  *code = 0;
  try {
    const std::vector<int> us(U, U + u);
    const plingam::DataMatrix data = to_data(X, n, d);
    const plingam::SearchResult r = workers > 1
                                        ? plingam::search_causal_order_parallel(data, std::span<const int>(us), workers)
                                        : plingam::search_causal_order(data, std::span<const int>(us));
    *chosen_out = r.chosen;
    for (std::size_t i = 0; i < r.scores.scores.size(); ++i) scores_out[i] = r.scores.scores[i];
    return 0;
  } catch (const plingam::Error& e) {
    return fail(e, code, row, col);
  }
}

}  // extern "C"
