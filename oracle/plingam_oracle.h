/*
 * plingam_oracle.h — CPU restatement of the reference DirectLiNGAM hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker, not the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load it. The product path (paper_2403_03772_b200) never links it.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/proj). The reference itself cannot be compiled here: it needs
 * Eigen3 >= 3.3 (proj/CMakeLists.txt:19, proj/src/kernels.cpp:3), which is absent
 * from this image and from the GPU box, so its Eigen packet exp/log1p are restated
 * with glibc exp/log1p. Parity of *orders* is pinned by the reference tests' known
 * answers (proj/tests/test_kernels.cpp, test_ordering.cpp); bit-level parity of
 * scores against Eigen is unpinned.
 *
 * Build: oracle/Makefile (gcc -O3 -ffp-contract=off, no -march: the reference's
 * own flags, proj/CMakeLists.txt:11-15).
 */
#ifndef PLINGAM_ORACLE_H
#define PLINGAM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status convention shared with the product C-ABI: code 0 = ok, otherwise
 * 1 + ordinal of plingam::ErrorCode (proj/include/plingam/error.hpp:10-27). */
typedef struct orc_status {
  int32_t code;
  int64_t row;
  int64_t col;
  char msg[256];
} orc_status;

enum {
  ORC_OK = 0,
  ORC_NonFinite = 1,
  ORC_ZeroVariance = 2,
  ORC_TooFewSamples = 3,
  ORC_TooShort = 4,
  ORC_LengthMismatch = 5,
  ORC_DimensionMismatch = 6,
  ORC_EmptyCandidates = 7,
  ORC_SingularDesign = 8,
  ORC_InsufficientRows = 9,
  ORC_UnstableSystem = 10,
  ORC_OutOfRange = 11,
  ORC_InvalidIndex = 12
};

/* ---- kernels (proj/src/kernels.cpp) ---- */
double orc_gaussian_entropy(void);                                   /* kernels.cpp:9 */
double orc_mean(const double* x, int64_t n);                          /* kernels.cpp:44-48 */
double orc_variance_pop_given_mean(const double* x, int64_t n, double m); /* :50-57 */
double orc_variance_pop(const double* x, int64_t n);                  /* :59-61 */
double orc_std_pop(const double* x, int64_t n);                       /* :63 */
double orc_covariance_pop_given_means(const double* x, const double* y, int64_t n,
                                      double mx, double my);          /* :65-75 */
double orc_covariance_pop(const double* x, const double* y, int64_t n); /* :77-79 */
double orc_log_cosh(double u);                                        /* :87-90 */
int orc_standardize(const double* x, int64_t n, double* out, orc_status* st);   /* :92-104 */
int orc_residual(const double* xi, const double* xj, int64_t n, double* out,
                 orc_status* st);                                     /* :106-121 */
double orc_entropy_approx(const double* u, int64_t n);                /* :123-132 */
int orc_entropy_of_normalized(const double* r, int64_t n, double* out, orc_status* st); /* :134-148 */
int orc_diff_mutual_info(const double* xi_std, const double* xj_std, const double* ri_j,
                         const double* rj_i, int64_t n, double* out, orc_status* st); /* :150-159 */

/* ---- data model (proj/src/types.cpp) ---- */
/* X is column-major n x d with leading dimension ld (>= n). */
int orc_validate(const double* X, int64_t n, int32_t d, int64_t ld, orc_status* st); /* types.cpp:21-47 */

/* ---- ordering (proj/src/ordering.cpp) ---- */
/* scores: d doubles, -inf for non-candidates. workers: 1 = sequential path
 * (ordering.cpp:166-168); >1 = static contiguous thread partition (:170-176).
 * fast != 0 evaluates every unordered pair once and uses the exact antisymmetry
 * mi(q,p) == -mi(p,q) (test_kernels.cpp:137-149); bit-identical, 2x cheaper. */
int orc_search_causal_order(const double* X, int64_t n, int32_t d, int64_t ld, const int32_t* U,
                            int32_t u, int32_t workers, int32_t fast, int32_t* chosen,
                            double* scores, orc_status* st);
/* out: n x r column-major (ld = n) */
int orc_regress_out(const double* X, int64_t n, int32_t d, int64_t ld, int32_t exog,
                    const int32_t* remaining, int32_t r, double* out, orc_status* st); /* :178-211 */
/* Full recursive order (ordering.cpp:213-244). max_rounds < 0 runs all d-1 rounds;
 * otherwise stops after max_rounds rounds (order_out holds that many entries) — used
 * to time a bounded prefix for the CPU baseline. round_scores (optional, may be NULL)
 * receives d doubles per executed round. */
int orc_causal_order(const double* X, int64_t n, int32_t d, int64_t ld, int32_t parallel,
                     int32_t workers, int32_t fast, int32_t max_rounds, int32_t* order_out,
                     double* round_scores, orc_status* st);

/* Full order by exact pruned rounds (the product's branch and bound on k, restated): same
 * order and winning k as orc_causal_order (tested), a few % of the pair evaluations.
 * winner_k (optional): d - 1 doubles, the k of each round's chosen variable; second_k
 * (optional): d - 1 doubles, a lower bound of the runner-up's k (exact when the runner-up
 * row was fully evaluated, its partial k otherwise), so second_k - winner_k bounds the
 * round's best-vs-second gap from below (near-tie guard, SURVEY §7 hard part 1). Golden
 * generation on valid data; error paths are not reproduced. */
int orc_causal_order_pruned(const double* X, int64_t n, int32_t d, int64_t ld, int32_t workers,
                            int32_t* order_out, double* winner_k, double* second_k, int64_t* pairs_evaluated,
                            orc_status* st);

/* ---- adjacency weights (proj/src/direct_lingam.cpp:46-70) ----
 * Per-target least squares on centred data via column-pivoted Householder QR
 * (Eigen::ColPivHouseholderQR); B is d x d column-major, B[target + d*pred].
 * used_pinv is set when a predecessor design is rank deficient; the
 * minimum-norm solution is then returned (Eigen::CompleteOrthogonalDecomposition). */
int orc_fit_weights(const double* X, int64_t n, int32_t d, int64_t ld, const int32_t* order,
                    double* B, int32_t* used_pinv, orc_status* st);

/* orc_fit_weights restricted to the targets at the listed order positions (rows of the
 * other targets stay zero): per-target spot checks at sizes where the full per-target
 * route would take hours. */
int orc_fit_weights_targets(const double* X, int64_t n, int32_t d, int64_t ld, const int32_t* order,
                            const int32_t* positions, int32_t npos, double* B, int32_t* used_pinv, orc_status* st);

/* The same weights from ONE Householder QR of the order-permuted centred design (every
 * predecessor regression is a prefix of it), rank-deficient columns in echelon form with
 * the minimum-norm correction (see the .c). O(n d^2) instead of the per-target O(n d^3):
 * the large-d reference, cross-checked against orc_fit_weights at small d.
 * n_dependent (optional): number of columns without a reflector. */
int orc_fit_weights_prefix(const double* X, int64_t n, int32_t d, int64_t ld, const int32_t* order,
                           int32_t nthreads, double* B, int32_t* used_pinv, int32_t* n_dependent,
                           orc_status* st);

/* ---- benchmark inputs without the product library (simgen_oracle.c; bench.py's reference
 * arm). Same bits as the package's generators (host/simgen.cpp). W is d x d column-major,
 * W[v + d*j] = weight of parent j in x_v; order = causal order; X is n x d column-major.
 * kind: 0 uniform(lo, hi), 1 Laplace(scale hi), 2 Student-t3 (scale hi), 3 N(lo, hi^2). */
int orc_gen_two_level_dag(int32_t d, uint64_t seed, double edge_prob, double* W, int32_t* order);
int orc_gen_sparse_dag(int32_t d, double avg_parents, uint64_t seed, double wmin, double wmax, double* W,
                       int32_t* order);
int orc_sample_lingam(const double* W, const int32_t* order, int32_t d, int64_t n, uint64_t seed, int32_t kind,
                      double lo, double hi, double* X);

#ifdef __cplusplus
}
#endif
#endif
