/*
 * plingam_oracle.c — CPU restatement of the reference DirectLiNGAM hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see plingam_oracle.h): the checker for the CUDA
 * product, and the CPU baseline timed beside it. Never linked by the product.
 *
 * Restates, function by function (paths relative to /root/reference/proj):
 *   src/kernels.cpp:16-159   moments, standardize, residual, entropy approximation
 *   src/types.cpp:21-47      validate
 *   src/ordering.cpp:16-244  search round, thread partition, argmax, regress_out, loop
 *   src/direct_lingam.cpp:46-70  per-target QR weights
 * Compiled with -O3 -ffp-contract=off and no -march, as the reference
 * (proj/CMakeLists.txt:11-15), so products and sums round exactly as written.
 * Eigen's ArrayXd exp/log1p (kernels.cpp:22-24) are replaced by glibc exp/log1p.
 */
#include "plingam_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* kernels.hpp:17 */
static const double kK1 = 79.047;
static const double kK2 = 7.4129;
static const double kGamma = 0.37457;
static const double kLn2 = 0.69314718055994530942; /* std::numbers::ln2 */
static const double kPi = 3.14159265358979323846;  /* std::numbers::pi */

static int set_status(orc_status* st, int32_t code, int64_t row, int64_t col, const char* fmt,
                      ...) {
  if (st) {
    st->code = code;
    st->row = row;
    st->col = col;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(st->msg, sizeof(st->msg), fmt, ap);
    va_end(ap);
  }
  return code;
}

static int ok(orc_status* st) {
  if (st) {
    st->code = 0;
    st->row = -1;
    st->col = -1;
    st->msg[0] = '\0';
  }
  return 0;
}

/* kernels.cpp:9 — kGaussianEntropy = 0.5 * (1 + log(2 pi)) */
double orc_gaussian_entropy(void) { return 0.5 * (1.0 + log(2.0 * kPi)); }

/* kernels.cpp:44-48 — strictly left-to-right sum, then divide by n */
double orc_mean(const double* x, int64_t n) {
  double s = 0.0;
  for (int64_t t = 0; t < n; ++t) s += x[t];
  return s / (double)n;
}

/* kernels.cpp:50-57 */
double orc_variance_pop_given_mean(const double* x, int64_t n, double m) {
  double s = 0.0;
  for (int64_t t = 0; t < n; ++t) {
    const double dv = x[t] - m;
    s += dv * dv;
  }
  return s / (double)n;
}

/* kernels.cpp:59-61 */
double orc_variance_pop(const double* x, int64_t n) {
  return orc_variance_pop_given_mean(x, n, orc_mean(x, n));
}

/* kernels.cpp:63 */
double orc_std_pop(const double* x, int64_t n) { return sqrt(orc_variance_pop(x, n)); }

/* kernels.cpp:65-75 */
double orc_covariance_pop_given_means(const double* x, const double* y, int64_t n, double mx,
                                      double my) {
  double s = 0.0;
  for (int64_t t = 0; t < n; ++t) s += (x[t] - mx) * (y[t] - my);
  return s / (double)n;
}

/* kernels.cpp:77-79 */
double orc_covariance_pop(const double* x, const double* y, int64_t n) {
  return orc_covariance_pop_given_means(x, y, n, orc_mean(x, n), orc_mean(y, n));
}

/* kernels.cpp:81-85 — out = xi - slope * xj (multiply, then subtract; no FMA) */
static void residual_into(const double* xi, const double* xj, int64_t n, double slope,
                          double* out) {
  for (int64_t t = 0; t < n; ++t) out[t] = xi[t] - slope * xj[t];
}

/* kernels.cpp:87-90 — association (a + log1p(exp(-2a))) - ln2 */
double orc_log_cosh(double u) {
  const double a = fabs(u);
  return a + log1p(exp(-2.0 * a)) - kLn2;
}

/* kernels.cpp:16-34 — lc_t = |u_t| + (log1p(exp(-2|u_t|)) - ln2) (Eigen `lc += expr`),
 * pdf_t = u_t * exp(-0.5 * u_t^2); two left-to-right sums. */
static void entropy_means(const double* u, int64_t n, double scale, int scaled, double* mean_lc,
                          double* mean_pdf) {
  double acc_lc = 0.0;
  double acc_pdf = 0.0;
  for (int64_t t = 0; t < n; ++t) {
    const double v = scaled ? u[t] / scale : u[t]; /* kernels.cpp:143 scratch = r / sd */
    const double a = fabs(v);
    const double lc = a + (log1p(exp(-2.0 * a)) - kLn2);
    const double sq = v * v;
    const double pdf = v * exp(-0.5 * sq);
    acc_lc += lc;
    acc_pdf += pdf;
  }
  *mean_lc = acc_lc / (double)n;
  *mean_pdf = acc_pdf / (double)n;
}

/* kernels.cpp:36-40 — ((kG - (k1*t1)*t1) - (k2*t2)*t2) */
static double entropy_from_means(double mean_lc, double mean_pdf) {
  const double t1 = mean_lc - kGamma;
  const double t2 = mean_pdf;
  return orc_gaussian_entropy() - kK1 * t1 * t1 - kK2 * t2 * t2;
}

/* kernels.cpp:92-104 */
int orc_standardize(const double* x, int64_t n, double* out, orc_status* st) {
  if (n < 2) return set_status(st, ORC_TooShort, -1, -1, "standardize: need at least 2 samples");
  const double m = orc_mean(x, n);
  const double sd = orc_std_pop(x, n);
  if (sd == 0.0) return set_status(st, ORC_ZeroVariance, -1, -1, "standardize: constant input");
  for (int64_t t = 0; t < n; ++t) out[t] = (x[t] - m) / sd;
  return ok(st);
}

/* kernels.cpp:106-121 */
int orc_residual(const double* xi, const double* xj, int64_t n, double* out, orc_status* st) {
  if (n < 2) return set_status(st, ORC_TooShort, -1, -1, "residual: need at least 2 samples");
  const double var_j = orc_variance_pop(xj, n);
  if (var_j == 0.0)
    return set_status(st, ORC_ZeroVariance, -1, -1, "residual: regressor has zero variance");
  const double slope = orc_covariance_pop(xi, xj, n) / var_j;
  residual_into(xi, xj, n, slope, out);
  return ok(st);
}

/* kernels.cpp:123-132 */
double orc_entropy_approx(const double* u, int64_t n) {
  double mlc, mpdf;
  entropy_means(u, n, 1.0, 0, &mlc, &mpdf);
  return entropy_from_means(mlc, mpdf);
}

/* kernels.cpp:134-148 — sd two-pass, scratch = r / sd (not re-centred) */
int orc_entropy_of_normalized(const double* r, int64_t n, double* out, orc_status* st) {
  const double sd = orc_std_pop(r, n);
  if (sd == 0.0)
    return set_status(st, ORC_ZeroVariance, -1, -1,
                      "entropy_of_normalized: zero residual (exactly collinear pair)");
  double mlc, mpdf;
  entropy_means(r, n, sd, 1, &mlc, &mpdf);
  *out = entropy_from_means(mlc, mpdf);
  return ok(st);
}

/* kernels.cpp:150-159 */
int orc_diff_mutual_info(const double* xi_std, const double* xj_std, const double* ri_j,
                         const double* rj_i, int64_t n, double* out, orc_status* st) {
  double e1, e2;
  int rc;
  const double hj = orc_entropy_approx(xj_std, n);
  if ((rc = orc_entropy_of_normalized(ri_j, n, &e1, st))) return rc;
  const double hi = orc_entropy_approx(xi_std, n);
  if ((rc = orc_entropy_of_normalized(rj_i, n, &e2, st))) return rc;
  const double favor_i = hj + e1;
  const double favor_j = hi + e2;
  *out = favor_i - favor_j;
  return ok(st);
}

/* types.cpp:21-47 — column by column: non-finite scan first, then zero variance */
int orc_validate(const double* X, int64_t n, int32_t d, int64_t ld, orc_status* st) {
  if (d < 1) return set_status(st, ORC_DimensionMismatch, -1, -1, "validate: need at least 1 variable");
  if (n < 2) return set_status(st, ORC_TooFewSamples, -1, -1, "validate: need at least 2 samples");
  for (int32_t j = 0; j < d; ++j) {
    const double* c = X + (int64_t)j * ld;
    for (int64_t i = 0; i < n; ++i) {
      if (!isfinite(c[i]))
        return set_status(st, ORC_NonFinite, i, j,
                          "validate: non-finite entry at row %lld, column x%d", (long long)i, j);
    }
    if (orc_variance_pop(c, n) == 0.0)
      return set_status(st, ORC_ZeroVariance, -1, j, "validate: column x%d has zero variance", j);
  }
  return ok(st);
}

/* ------------------------------------------------------------------ ordering */

static int cmp_int(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* ordering.cpp:16-33 */
static int sorted_candidates(int32_t d, const int32_t* U, int32_t u, int32_t* out,
                             orc_status* st) {
  if (u <= 0)
    return set_status(st, ORC_EmptyCandidates, -1, -1, "search_causal_order: empty candidate set");
  memcpy(out, U, sizeof(int32_t) * (size_t)u);
  qsort(out, (size_t)u, sizeof(int32_t), cmp_int);
  for (int32_t p = 0; p < u; ++p) {
    if (out[p] < 0 || out[p] >= d)
      return set_status(st, ORC_InvalidIndex, -1, out[p],
                        "search_causal_order: candidate index out of range");
    if (p > 0 && out[p] == out[p - 1])
      return set_status(st, ORC_InvalidIndex, -1, out[p],
                        "search_causal_order: duplicate candidate index");
  }
  return ok(st);
}

/* ordering.cpp:40-45 RoundCache */
typedef struct {
  int64_t n;
  int32_t u;
  double* std_cols; /* u x n */
  double* col_entropy;
  double* col_mean;
  double* col_var;
} round_cache;

static void free_cache(round_cache* c) {
  free(c->std_cols);
  free(c->col_entropy);
  free(c->col_mean);
  free(c->col_var);
}

/* ordering.cpp:47-70 */
static int build_cache(const double* X, int64_t n, int64_t ld, const int32_t* u, int32_t nu,
                       round_cache* c, orc_status* st) {
  c->n = n;
  c->u = nu;
  c->std_cols = (double*)malloc(sizeof(double) * (size_t)nu * (size_t)n);
  c->col_entropy = (double*)malloc(sizeof(double) * (size_t)nu);
  c->col_mean = (double*)malloc(sizeof(double) * (size_t)nu);
  c->col_var = (double*)malloc(sizeof(double) * (size_t)nu);
  for (int32_t p = 0; p < nu; ++p) {
    double* z = c->std_cols + (int64_t)p * n;
    orc_status s2;
    int rc = orc_standardize(X + (int64_t)u[p] * ld, n, z, &s2);
    if (rc == ORC_ZeroVariance)
      return set_status(st, ORC_ZeroVariance, -1, u[p],
                        "search_causal_order: column %d has zero variance", u[p]);
    if (rc) {
      if (st) *st = s2;
      return rc;
    }
    c->col_entropy[p] = orc_entropy_approx(z, n);
    c->col_mean[p] = orc_mean(z, n);
    c->col_var[p] = orc_variance_pop_given_mean(z, n, c->col_mean[p]);
  }
  return ok(st);
}

/* The shared part of candidate_score (ordering.cpp:83-94): mi_diff for candidate at
 * position p against position q, both residual directions, one shared covariance. */
static int pair_mi(const round_cache* c, int32_t p, int32_t q, double* ri_j, double* rj_i,
                   double* mi, orc_status* st) {
  const int64_t n = c->n;
  const double* xi = c->std_cols + (int64_t)p * n;
  const double* xj = c->std_cols + (int64_t)q * n;
  const double cov = orc_covariance_pop_given_means(xi, xj, n, c->col_mean[p], c->col_mean[q]);
  residual_into(xi, xj, n, cov / c->col_var[q], ri_j);
  residual_into(xj, xi, n, cov / c->col_var[p], rj_i);
  double e1, e2;
  int rc;
  if ((rc = orc_entropy_of_normalized(ri_j, n, &e1, st))) return rc;
  const double favor_i = c->col_entropy[q] + e1;
  if ((rc = orc_entropy_of_normalized(rj_i, n, &e2, st))) return rc;
  const double favor_j = c->col_entropy[p] + e2;
  *mi = favor_i - favor_j;
  return 0;
}

/* std::min(0.0, mi) == (mi < 0.0) ? mi : 0.0 */
static inline double clip0(double mi) { return (mi < 0.0) ? mi : 0.0; }

/* ordering.cpp:78-99 */
static int candidate_score(const round_cache* c, int32_t p, double* ri_j, double* rj_i,
                           double* score, orc_status* st) {
  double k = 0.0;
  for (int32_t q = 0; q < c->u; ++q) {
    if (q == p) continue;
    double mi;
    int rc = pair_mi(c, p, q, ri_j, rj_i, &mi, st);
    if (rc) return rc;
    const double cl = clip0(mi);
    k += cl * cl;
  }
  *score = -k;
  return 0;
}

typedef struct {
  const round_cache* cache;
  const double* mi_full; /* fast path: u x u antisymmetric matrix, or NULL */
  double* pos_scores;    /* per position */
  int32_t lo, hi;
  int rc;
  orc_status st;
} chunk_job;

static void* run_chunk(void* arg) {
  chunk_job* job = (chunk_job*)arg;
  const round_cache* c = job->cache;
  job->rc = 0;
  if (job->mi_full) {
    for (int32_t p = job->lo; p < job->hi; ++p) {
      double k = 0.0;
      for (int32_t q = 0; q < c->u; ++q) {
        if (q == p) continue;
        const double cl = clip0(job->mi_full[(int64_t)p * c->u + q]);
        k += cl * cl;
      }
      job->pos_scores[p] = -k;
    }
    return NULL;
  }
  double* ri_j = (double*)malloc(sizeof(double) * (size_t)c->n);
  double* rj_i = (double*)malloc(sizeof(double) * (size_t)c->n);
  for (int32_t p = job->lo; p < job->hi; ++p) {
    int rc = candidate_score(c, p, ri_j, rj_i, &job->pos_scores[p], &job->st);
    if (rc) {
      job->rc = rc;
      break;
    }
  }
  free(ri_j);
  free(rj_i);
  return NULL;
}

/* Fast-exact: mi for every unordered pair p<q once; mi(q,p) = -mi(p,q) exactly because
 * the covariance is symmetric bit for bit and IEEE subtraction is antisymmetric
 * (test_kernels.cpp:137-149). Errors are reproduced in sequential order: the first
 * failing (p, q) in p-major, q-ascending order, as candidate_score would hit it. */
typedef struct {
  const round_cache* cache;
  double* mi_full;
  int32_t p_lo, p_hi;
  int rc;
  int32_t err_p, err_q;
  orc_status st;
} tri_job;

static void* run_tri(void* arg) {
  tri_job* job = (tri_job*)arg;
  const round_cache* c = job->cache;
  double* ri_j = (double*)malloc(sizeof(double) * (size_t)c->n);
  double* rj_i = (double*)malloc(sizeof(double) * (size_t)c->n);
  job->rc = 0;
  job->err_p = job->err_q = -1;
  for (int32_t p = job->p_lo; p < job->p_hi; ++p) {
    for (int32_t q = p + 1; q < c->u; ++q) {
      double mi;
      orc_status s2;
      int rc = pair_mi(c, p, q, ri_j, rj_i, &mi, &s2);
      if (rc) {
        if (!job->rc) {
          job->rc = rc;
          job->st = s2;
          job->err_p = p;
          job->err_q = q;
        }
        mi = 0.0;
      }
      job->mi_full[(int64_t)p * c->u + q] = mi;
      job->mi_full[(int64_t)q * c->u + p] = -mi;
    }
  }
  free(ri_j);
  free(rj_i);
  return NULL;
}

static int run_threads(void* jobs, size_t job_size, int32_t nthreads, void* (*fn)(void*)) {
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int32_t c = 1; c < nthreads; ++c)
    pthread_create(&th[c], NULL, fn, (char*)jobs + job_size * (size_t)c);
  fn(jobs);
  for (int32_t c = 1; c < nthreads; ++c) pthread_join(th[c], NULL);
  free(th);
  return 0;
}

/* ordering.cpp:101-162 */
static int search_impl(const double* X, int64_t n, int32_t d, int64_t ld, const int32_t* U,
                       int32_t nu, int32_t workers, int32_t fast, int32_t* chosen,
                       double* scores, orc_status* st) {
  int32_t* u = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nu > 0 ? nu : 1));
  int rc = sorted_candidates(d, U, nu, u, st);
  if (rc) {
    free(u);
    return rc;
  }
  for (int32_t j = 0; j < d; ++j) scores[j] = -INFINITY;
  if (nu == 1) { /* ordering.cpp:107-110 */
    scores[u[0]] = 0.0;
    *chosen = u[0];
    free(u);
    return ok(st);
  }
  round_cache cache;
  memset(&cache, 0, sizeof(cache));
  rc = build_cache(X, n, ld, u, nu, &cache, st);
  if (rc) {
    free_cache(&cache);
    free(u);
    return rc;
  }
  /* ordering.cpp:114-116: nthreads = clamp(workers, 1, |U|) */
  int32_t nthreads = workers < 1 ? 1 : workers;
  if (nthreads > nu) nthreads = nu;
  double* pos_scores = (double*)malloc(sizeof(double) * (size_t)nu);
  double* mi_full = NULL;

  if (fast) {
    mi_full = (double*)calloc((size_t)nu * (size_t)nu, sizeof(double));
    /* balance the triangle: rows p cost (nu-1-p); split rows so chunks have ~equal pairs */
    tri_job* tj = (tri_job*)calloc((size_t)nthreads, sizeof(tri_job));
    const double total = 0.5 * (double)nu * (double)(nu - 1);
    int32_t p = 0;
    for (int32_t c = 0; c < nthreads; ++c) {
      tj[c].cache = &cache;
      tj[c].mi_full = mi_full;
      tj[c].p_lo = p;
      const double target = total * (double)(c + 1) / (double)nthreads;
      double acc = 0.5 * (double)p * (double)(2 * nu - p - 1);
      while (p < nu && (c == nthreads - 1 || acc < target)) {
        acc += (double)(nu - 1 - p);
        ++p;
      }
      tj[c].p_hi = p;
    }
    run_threads(tj, sizeof(tri_job), nthreads, run_tri);
    /* first error in sequential order: lowest (min(p,q) by candidate p sweep). Candidate
     * p meets pair {p,q} at q; candidate_score(p) visits q ascending, so the sequential
     * path fails at the smallest p that belongs to any failing pair, at its smallest
     * failing partner. Every failing pair has both members as failing candidates. */
    int32_t best_p = -1;
    orc_status best_st;
    memset(&best_st, 0, sizeof(best_st));
    for (int32_t c = 0; c < nthreads; ++c) {
      if (tj[c].rc && (best_p < 0 || tj[c].err_p < best_p)) {
        best_p = tj[c].err_p;
        best_st = tj[c].st;
      }
    }
    free(tj);
    if (best_p >= 0) {
      if (st) *st = best_st;
      rc = best_st.code;
      goto done;
    }
  }
  {
    chunk_job* jobs = (chunk_job*)calloc((size_t)nthreads, sizeof(chunk_job));
    const int32_t base = nu / nthreads, rem = nu % nthreads;
    for (int32_t c = 0; c < nthreads; ++c) {
      jobs[c].cache = &cache;
      jobs[c].mi_full = mi_full;
      jobs[c].pos_scores = pos_scores;
      jobs[c].lo = c * base + (c < rem ? c : rem); /* ordering.cpp:119 chunk_begin */
      jobs[c].hi = (c + 1) * base + (c + 1 < rem ? c + 1 : rem);
    }
    run_threads(jobs, sizeof(chunk_job), nthreads, run_chunk);
    for (int32_t c = 0; c < nthreads; ++c) { /* lowest chunk's error, ordering.cpp:147-151 */
      if (jobs[c].rc) {
        if (st) *st = jobs[c].st;
        rc = jobs[c].rc;
        free(jobs);
        goto done;
      }
    }
    free(jobs);
  }
  for (int32_t p = 0; p < nu; ++p) scores[u[p]] = pos_scores[p];
  {
    /* ordering.cpp:154-160: strict '>' over ascending candidates, lowest index wins */
    int32_t best = 0;
    for (int32_t p = 1; p < nu; ++p)
      if (scores[u[p]] > scores[u[best]]) best = p;
    *chosen = u[best];
  }
  rc = ok(st);
done:
  free(mi_full);
  free(pos_scores);
  free_cache(&cache);
  free(u);
  return rc;
}

/* ordering.cpp:166-176 */
int orc_search_causal_order(const double* X, int64_t n, int32_t d, int64_t ld, const int32_t* U,
                            int32_t u, int32_t workers, int32_t fast, int32_t* chosen,
                            double* scores, orc_status* st) {
  if (workers < 1)
    return set_status(st, ORC_OutOfRange, -1, -1,
                      "search_causal_order_parallel: workers must be >= 1");
  return search_impl(X, n, d, ld, U, u, workers, fast, chosen, scores, st);
}

/* ordering.cpp:178-211 (+ kernels.cpp:106-121 residual): raw working columns, means
 * and variance recomputed from scratch for every remaining column. */
int orc_regress_out(const double* X, int64_t n, int32_t d, int64_t ld, int32_t exog,
                    const int32_t* remaining, int32_t r, double* out, orc_status* st) {
  if (exog < 0 || exog >= d)
    return set_status(st, ORC_InvalidIndex, -1, exog, "regress_out: exog index out of range");
  const double* xm = X + (int64_t)exog * ld;
  for (int32_t p = 0; p < r; ++p) {
    const int32_t c = remaining[p];
    if (c < 0 || c >= d)
      return set_status(st, ORC_InvalidIndex, -1, c, "regress_out: remaining index out of range");
    if (c == exog)
      return set_status(st, ORC_InvalidIndex, -1, c, "regress_out: exog cannot appear in remaining");
    orc_status s2;
    int rc = orc_residual(X + (int64_t)c * ld, xm, n, out + (int64_t)p * n, &s2);
    if (rc == ORC_ZeroVariance)
      return set_status(st, ORC_ZeroVariance, -1, exog,
                        "regress_out: exogenous column %d has zero variance", exog);
    if (rc) {
      if (st) *st = s2;
      return rc;
    }
  }
  return ok(st);
}

/* ordering.cpp:213-244 */
int orc_causal_order(const double* X, int64_t n, int32_t d, int64_t ld, int32_t parallel,
                     int32_t workers, int32_t fast, int32_t max_rounds, int32_t* order_out,
                     double* round_scores, orc_status* st) {
  int rc = orc_validate(X, n, d, ld, st);
  if (rc) return rc;
  if (workers < 1) return set_status(st, ORC_OutOfRange, -1, -1, "causal_order: workers must be >= 1");
  double* working = (double*)malloc(sizeof(double) * (size_t)n * (size_t)d);
  for (int32_t j = 0; j < d; ++j)
    memcpy(working + (int64_t)j * n, X + (int64_t)j * ld, sizeof(double) * (size_t)n);
  int32_t* u = (int32_t*)malloc(sizeof(int32_t) * (size_t)d);
  int32_t* rem = (int32_t*)malloc(sizeof(int32_t) * (size_t)d);
  double* scores = (double*)malloc(sizeof(double) * (size_t)d);
  double* res = (double*)malloc(sizeof(double) * (size_t)n * (size_t)(d > 1 ? d - 1 : 1));
  for (int32_t p = 0; p < d; ++p) u[p] = p;
  int32_t nu = d, pos = 0, rounds = 0;
  rc = 0;
  while (nu > 1) {
    if (max_rounds >= 0 && rounds >= max_rounds) break;
    int32_t chosen = -1;
    rc = search_impl(working, n, d, n, u, nu, parallel ? workers : 1, fast, &chosen, scores, st);
    if (rc) break;
    if (round_scores) memcpy(round_scores + (int64_t)rounds * d, scores, sizeof(double) * (size_t)d);
    int32_t nr = 0;
    for (int32_t p = 0; p < nu; ++p)
      if (u[p] != chosen) rem[nr++] = u[p];
    rc = orc_regress_out(working, n, d, n, chosen, rem, nr, res, st);
    if (rc) break;
    for (int32_t p = 0; p < nr; ++p)
      memcpy(working + (int64_t)rem[p] * n, res + (int64_t)p * n, sizeof(double) * (size_t)n);
    order_out[pos++] = chosen;
    memcpy(u, rem, sizeof(int32_t) * (size_t)nr);
    nu = nr;
    ++rounds;
  }
  if (!rc && nu == 1) order_out[pos++] = u[0];
  free(working);
  free(u);
  free(rem);
  free(scores);
  free(res);
  return rc ? rc : ok(st);
}

/* ------------------------------------------------------------ exact pruned order */
/* The product's pruned rounds (prune_kernels.cu) restated on the CPU, used to produce full
 * golden orders for the largest configs (C3, C5) in minutes instead of days. Each round
 * evaluates pair_mi only for the pairs a branch and bound on k needs: R = 3 rows with the
 * lowest predicted k get full rows (k* = min of their exact k), every other row its T = 2
 * strongest predicted partners, then rows whose partial k is still <= k* (1 + 1e-9) their
 * strongest partners up to 5% and 25% of the row, then the survivors full rows. A row's
 * partial k is a sum of a subset of its non-negative terms, so pruned rows cannot win; the
 * winner's k is summed exactly as candidate_score (q ascending) from the same pair_mi
 * values, so order and winning k equal the fast/faithful modes' (tested bit for bit).
 * Predictions: the last evaluated min(0, mi)^2 of each variable pair (round 0 evaluates
 * every pair). Error paths are not reproduced (golden generation on valid data only). */
typedef struct {
  const round_cache* cache;
  double* mi_full;
  const int32_t* pp;
  const int32_t* qq;
  int64_t lo, hi;
  int rc;
  orc_status st;
} list_job;

static void* run_list(void* arg) {
  list_job* job = (list_job*)arg;
  const round_cache* c = job->cache;
  double* ri_j = (double*)malloc(sizeof(double) * (size_t)c->n);
  double* rj_i = (double*)malloc(sizeof(double) * (size_t)c->n);
  job->rc = 0;
  for (int64_t k = job->lo; k < job->hi && !job->rc; ++k) {
    const int32_t p = job->pp[k], q = job->qq[k];
    double mi;
    int rc = pair_mi(c, p, q, ri_j, rj_i, &mi, &job->st);
    if (rc) {
      job->rc = rc;
      break;
    }
    job->mi_full[(int64_t)p * c->u + q] = mi;
    job->mi_full[(int64_t)q * c->u + p] = -mi;
  }
  free(ri_j);
  free(rj_i);
  return NULL;
}

typedef struct {
  int32_t* pp;
  int32_t* qq;
  int64_t n, cap;
  uint8_t* queued; /* u x u */
} pair_list;

static void list_add(pair_list* L, int32_t u, int32_t p, int32_t q, const double* mi_full) {
  const int32_t a = p < q ? p : q, b = p < q ? q : p;
  if (a == b || L->queued[(int64_t)a * u + b] || mi_full[(int64_t)a * u + b] == mi_full[(int64_t)a * u + b])
    return;
  L->queued[(int64_t)a * u + b] = 1;
  if (L->n == L->cap) {
    L->cap = L->cap ? 2 * L->cap : 1024;
    L->pp = (int32_t*)realloc(L->pp, sizeof(int32_t) * (size_t)L->cap);
    L->qq = (int32_t*)realloc(L->qq, sizeof(int32_t) * (size_t)L->cap);
  }
  L->pp[L->n] = a;
  L->qq[L->n] = b;
  ++L->n;
}

static int eval_list(const round_cache* c, double* mi_full, pair_list* L, int32_t nthreads, int64_t* evaluated,
                     orc_status* st) {
  if (L->n == 0) return 0;
  list_job* jobs = (list_job*)calloc((size_t)nthreads, sizeof(list_job));
  for (int32_t t = 0; t < nthreads; ++t) {
    jobs[t].cache = c;
    jobs[t].mi_full = mi_full;
    jobs[t].pp = L->pp;
    jobs[t].qq = L->qq;
    jobs[t].lo = L->n * t / nthreads;
    jobs[t].hi = L->n * (t + 1) / nthreads;
  }
  run_threads(jobs, sizeof(list_job), nthreads, run_list);
  int rc = 0;
  for (int32_t t = 0; t < nthreads && !rc; ++t)
    if (jobs[t].rc) {
      rc = jobs[t].rc;
      if (st) *st = jobs[t].st;
    }
  free(jobs);
  for (int64_t k = 0; k < L->n; ++k) L->queued[(int64_t)L->pp[k] * c->u + L->qq[k]] = 0;
  *evaluated += L->n;
  L->n = 0;
  return rc;
}

/* k of position p over its evaluated partners, q ascending (candidate_score's order) */
static double partial_k(const double* mi_full, int32_t u, int32_t p) {
  double k = 0.0;
  for (int32_t q = 0; q < u; ++q) {
    if (q == p) continue;
    const double mi = mi_full[(int64_t)p * u + q];
    if (mi != mi) continue;
    const double cl = clip0(mi);
    k += cl * cl;
  }
  return k;
}

static const double* g_key_row; /* qsort context: predictions of the row being selected */
static int cmp_key_desc(const void* a, const void* b) {
  const int32_t qa = *(const int32_t*)a, qb = *(const int32_t*)b;
  const double ka = g_key_row[qa], kb = g_key_row[qb];
  if (ka != kb) return ka > kb ? -1 : 1;
  return (qa > qb) - (qa < qb);
}

int orc_causal_order_pruned(const double* X, int64_t n, int32_t d, int64_t ld, int32_t workers,
                            int32_t* order_out, double* winner_k, double* second_k, int64_t* pairs_evaluated,
                            orc_status* st) {
  int rc = orc_validate(X, n, d, ld, st);
  if (rc) return rc;
  if (workers < 1) workers = 1;
  const int32_t R = 3, T = 2;
  const double fracs[2] = {0.05, 0.25};
  double* working = (double*)malloc(sizeof(double) * (size_t)n * (size_t)d);
  for (int32_t j = 0; j < d; ++j)
    memcpy(working + (int64_t)j * n, X + (int64_t)j * ld, sizeof(double) * (size_t)n);
  int32_t* u = (int32_t*)malloc(sizeof(int32_t) * (size_t)d);
  int32_t* rem = (int32_t*)malloc(sizeof(int32_t) * (size_t)d);
  double* res = (double*)malloc(sizeof(double) * (size_t)n * (size_t)(d > 1 ? d - 1 : 1));
  double* KN = (double*)calloc((size_t)d * (size_t)d, sizeof(double));
  double* mi_full = (double*)malloc(sizeof(double) * (size_t)d * (size_t)d);
  double* kex = (double*)malloc(sizeof(double) * (size_t)d);
  double* key = (double*)malloc(sizeof(double) * (size_t)d);
  int32_t* state = (int32_t*)malloc(sizeof(int32_t) * (size_t)d);
  int32_t* cand = (int32_t*)malloc(sizeof(int32_t) * (size_t)d);
  pair_list L = {NULL, NULL, 0, 0, (uint8_t*)calloc((size_t)d * (size_t)d, 1)};
  int64_t evaluated = 0;
  for (int32_t p = 0; p < d; ++p) u[p] = p;
  int32_t nu = d, pos = 0, round = 0;
  rc = 0;
  while (nu > 1) {
    round_cache cache;
    memset(&cache, 0, sizeof(cache));
    rc = build_cache(working, n, n, u, nu, &cache, st);
    if (rc) {
      free_cache(&cache);
      break;
    }
    const int32_t nthreads = workers;
    for (int64_t i = 0; i < (int64_t)nu * nu; ++i) mi_full[i] = NAN;
    const int exhaustive = (round == 0 || nu <= 8);
    int32_t best = -1;
    if (exhaustive) {
      for (int32_t p = 0; p < nu; ++p)
        for (int32_t q = p + 1; q < nu; ++q) list_add(&L, nu, p, q, mi_full);
      rc = eval_list(&cache, mi_full, &L, nthreads, &evaluated, st);
      for (int32_t p = 0; p < nu; ++p) {
        kex[p] = partial_k(mi_full, nu, p);
        state[p] = 1;
      }
    } else {
      double* pk = key; /* predicted k per position */
      for (int32_t p = 0; p < nu; ++p) {
        double a = 0.0;
        for (int32_t q = 0; q < nu; ++q)
          if (q != p) a += KN[(int64_t)u[p] * d + u[q]];
        pk[p] = a;
        state[p] = 1;
      }
      for (int32_t r = 0; r < R && r < nu; ++r) { /* top: lowest predicted k, lowest position */
        int32_t b = -1;
        for (int32_t p = 0; p < nu; ++p)
          if (state[p] == 1 && (b < 0 || pk[p] < pk[b])) b = p;
        state[b] = 2;
      }
      for (int32_t p = 0; p < nu; ++p) {
        if (state[p] == 2) {
          for (int32_t q = 0; q < nu; ++q) list_add(&L, nu, p, q, mi_full);
        } else {
          int32_t nc = 0;
          for (int32_t q = 0; q < nu; ++q)
            if (q != p && state[q] != 2) cand[nc++] = q;
          for (int32_t q = 0; q < nu; ++q) key[q] = KN[(int64_t)u[p] * d + u[q]];
          g_key_row = key;
          qsort(cand, (size_t)nc, sizeof(int32_t), cmp_key_desc);
          for (int32_t i = 0; i < T && i < nc; ++i) list_add(&L, nu, p, cand[i], mi_full);
        }
      }
      if (!rc) rc = eval_list(&cache, mi_full, &L, nthreads, &evaluated, st);
      double kstar = INFINITY;
      for (int32_t p = 0; p < nu; ++p)
        if (state[p] == 2) {
          kex[p] = partial_k(mi_full, nu, p);
          if (kex[p] < kstar) kstar = kex[p];
        }
      const double thr = kstar * (1.0 + 1e-9);
      double prev = 0.0;
      for (int32_t stage = 0; stage <= 2 && !rc; ++stage) {
        for (int32_t p = 0; p < nu; ++p) {
          if (state[p] != 1) continue;
          if (partial_k(mi_full, nu, p) > thr) {
            state[p] = 0;
            continue;
          }
          if (stage == 2) { /* full row */
            for (int32_t q = 0; q < nu; ++q) list_add(&L, nu, p, q, mi_full);
            continue;
          }
          const int32_t m = (int32_t)((fracs[stage] - prev) * nu) > 0 ? (int32_t)((fracs[stage] - prev) * nu) : 1;
          int32_t nc = 0;
          for (int32_t q = 0; q < nu; ++q) {
            const double mi = mi_full[(int64_t)p * nu + q];
            if (q != p && mi != mi) cand[nc++] = q;
          }
          for (int32_t q = 0; q < nu; ++q) key[q] = KN[(int64_t)u[p] * d + u[q]];
          g_key_row = key;
          qsort(cand, (size_t)nc, sizeof(int32_t), cmp_key_desc);
          for (int32_t i = 0; i < m && i < nc; ++i) list_add(&L, nu, p, cand[i], mi_full);
        }
        if (stage < 2) prev = fracs[stage];
        rc = eval_list(&cache, mi_full, &L, nthreads, &evaluated, st);
      }
      for (int32_t p = 0; p < nu; ++p)
        if (state[p] == 1) kex[p] = partial_k(mi_full, nu, p);
    }
    free_cache(&cache);
    if (rc) break;
    for (int32_t p = 0; p < nu; ++p) /* ordering.cpp:154-160: lowest position on ties */
      if (state[p] >= 1 && (best < 0 || kex[p] < kex[best])) best = p;
    for (int32_t p = 0; p < nu; ++p) /* knowledge: evaluated pairs */
      for (int32_t q = 0; q < nu; ++q) {
        const double mi = mi_full[(int64_t)p * nu + q];
        if (q != p && mi == mi) {
          const double cl = clip0(mi);
          KN[(int64_t)u[p] * d + u[q]] = cl * cl;
        }
      }
    if (winner_k) winner_k[round] = kex[best];
    if (second_k) { /* runner-up: exact k of evaluated rows, the partial k (a lower bound) of pruned ones */
      double s2 = INFINITY;
      for (int32_t p = 0; p < nu; ++p) {
        if (p == best) continue;
        const double kp = state[p] >= 1 ? kex[p] : partial_k(mi_full, nu, p);
        if (kp < s2) s2 = kp;
      }
      second_k[round] = s2;
    }
    const int32_t chosen = u[best];
    int32_t nr = 0;
    for (int32_t p = 0; p < nu; ++p)
      if (u[p] != chosen) rem[nr++] = u[p];
    rc = orc_regress_out(working, n, d, n, chosen, rem, nr, res, st);
    if (rc) break;
    for (int32_t p = 0; p < nr; ++p)
      memcpy(working + (int64_t)rem[p] * n, res + (int64_t)p * n, sizeof(double) * (size_t)n);
    order_out[pos++] = chosen;
    memcpy(u, rem, sizeof(int32_t) * (size_t)nr);
    nu = nr;
    ++round;
  }
  if (!rc && nu == 1) order_out[pos++] = u[0];
  if (pairs_evaluated) *pairs_evaluated = evaluated;
  free(working);
  free(u);
  free(rem);
  free(res);
  free(KN);
  free(mi_full);
  free(kex);
  free(key);
  free(state);
  free(cand);
  free(L.pp);
  free(L.qq);
  free(L.queued);
  return rc ? rc : ok(st);
}

/* ------------------------------------------------------------------ weights */

/* Column-pivoted Householder QR of A (m x p, column-major, lda = m), in place, in the
 * manner of Eigen::ColPivHouseholderQR: pivot = remaining column of largest norm, norms
 * downdated and recomputed on cancellation; rank = #|R_kk| > eps * min(m,p) * |max pivot|.
 * hcoef receives the Householder scalars, perm the column permutation. */
static int32_t colpiv_qr(double* A, int64_t m, int32_t p, double* hcoef, int32_t* perm) {
  double* norms = (double*)malloc(sizeof(double) * (size_t)p);
  double* norms_direct = (double*)malloc(sizeof(double) * (size_t)p);
  for (int32_t j = 0; j < p; ++j) {
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) s += A[i + m * j] * A[i + m * j];
    norms[j] = norms_direct[j] = sqrt(s);
    perm[j] = j;
  }
  const int32_t k_max = (int32_t)(m < p ? m : p);
  double max_pivot = 0.0;
  for (int32_t k = 0; k < k_max; ++k) {
    int32_t big = k;
    for (int32_t j = k + 1; j < p; ++j)
      if (norms[j] > norms[big]) big = j;
    if (big != k) {
      for (int64_t i = 0; i < m; ++i) {
        const double t = A[i + m * k];
        A[i + m * k] = A[i + m * big];
        A[i + m * big] = t;
      }
      double t = norms[k]; norms[k] = norms[big]; norms[big] = t;
      t = norms_direct[k]; norms_direct[k] = norms_direct[big]; norms_direct[big] = t;
      int32_t ti = perm[k]; perm[k] = perm[big]; perm[big] = ti;
    }
    /* Householder vector for A[k:m, k] */
    double* col = A + m * k;
    double tail = 0.0;
    for (int64_t i = k + 1; i < m; ++i) tail += col[i] * col[i];
    double beta, tau;
    const double c0 = col[k];
    if (tail == 0.0) {
      tau = 0.0;
      beta = c0;
    } else {
      beta = sqrt(c0 * c0 + tail);
      if (c0 >= 0.0) beta = -beta;
      const double denom = c0 - beta;
      for (int64_t i = k + 1; i < m; ++i) col[i] /= denom;
      tau = (beta - c0) / beta;
    }
    col[k] = beta;
    hcoef[k] = tau;
    if (fabs(beta) > max_pivot) max_pivot = fabs(beta);
    /* apply H = I - tau v v^T (v[k]=1) to the trailing columns */
    for (int32_t j = k + 1; j < p; ++j) {
      double* cj = A + m * j;
      double s = cj[k];
      for (int64_t i = k + 1; i < m; ++i) s += col[i] * cj[i];
      s *= tau;
      cj[k] -= s;
      for (int64_t i = k + 1; i < m; ++i) cj[i] -= s * col[i];
      /* norm downdate (LAPACK xGEQPF style, as Eigen) */
      if (norms[j] != 0.0) {
        double temp = fabs(cj[k]) / norms[j];
        temp = (1.0 + temp) * (1.0 - temp);
        if (temp < 0.0) temp = 0.0;
        const double temp2 = temp * (norms[j] / norms_direct[j]) * (norms[j] / norms_direct[j]);
        if (temp2 <= sqrt(2.220446049250313e-16)) {
          double s2 = 0.0;
          for (int64_t i = k + 1; i < m; ++i) s2 += cj[i] * cj[i];
          norms_direct[j] = norms[j] = sqrt(s2);
        } else {
          norms[j] *= sqrt(temp);
        }
      }
    }
  }
  const double thr = 2.220446049250313e-16 * (double)k_max * max_pivot;
  int32_t rank = 0;
  for (int32_t k = 0; k < k_max; ++k)
    if (fabs(A[k + m * k]) > thr) ++rank;
  free(norms);
  free(norms_direct);
  return rank;
}

/* apply Q^T (from colpiv_qr) to b in place */
static void apply_qt(const double* A, int64_t m, int32_t kk, const double* hcoef, double* b) {
  for (int32_t k = 0; k < kk; ++k) {
    const double* v = A + m * k;
    double s = b[k];
    for (int64_t i = k + 1; i < m; ++i) s += v[i] * b[i];
    s *= hcoef[k];
    b[k] -= s;
    for (int64_t i = k + 1; i < m; ++i) b[i] -= s * v[i];
  }
}

/* Minimum-norm least squares for a rank-r design (Eigen CompleteOrthogonalDecomposition):
 * after A P = Q [R11 R12; 0 0], reduce [R11 R12] (r x p) to [T 0] Z by Householder
 * reflections from the right, then x = P Z^T [T^-1 (Q^T b)[0:r]; 0]. */
static void cod_solve(const double* Aqr, int64_t m, int32_t p, int32_t r, const int32_t* perm,
                      const double* qtb, double* x) {
  /* W = R[0:r, 0:p] (row-major r x p for row reflections) */
  double* W = (double*)calloc((size_t)(r > 0 ? r : 1) * (size_t)p, sizeof(double));
  for (int32_t i = 0; i < r; ++i)
    for (int32_t j = i; j < p; ++j) W[(int64_t)i * p + j] = Aqr[i + m * j];
  double* zv = (double*)calloc((size_t)(r > 0 ? r : 1) * (size_t)p, sizeof(double)); /* reflector vectors */
  double* ztau = (double*)calloc((size_t)(r > 0 ? r : 1), sizeof(double));
  for (int32_t i = r - 1; i >= 0; --i) {
    /* reflect row i entries {i, r..p-1} so that entries r..p-1 vanish */
    double* row = W + (int64_t)i * p;
    double tail = 0.0;
    for (int32_t j = r; j < p; ++j) tail += row[j] * row[j];
    if (tail == 0.0) continue;
    const double a0 = row[i];
    double beta = sqrt(a0 * a0 + tail);
    if (a0 >= 0.0) beta = -beta;
    const double denom = a0 - beta;
    double* v = zv + (int64_t)i * p;
    v[i] = 1.0;
    for (int32_t j = r; j < p; ++j) v[j] = row[j] / denom;
    ztau[i] = (beta - a0) / beta;
    /* apply to rows 0..i (row i gets [beta, 0...]) */
    for (int32_t rr = 0; rr <= i; ++rr) {
      double* w = W + (int64_t)rr * p;
      double s = w[i];
      for (int32_t j = r; j < p; ++j) s += w[j] * v[j];
      s *= ztau[i];
      w[i] -= s;
      for (int32_t j = r; j < p; ++j) w[j] -= s * v[j];
    }
  }
  /* solve T y = qtb[0:r] (T upper triangular r x r in W[:, 0:r]) */
  double* y = (double*)calloc((size_t)p, sizeof(double));
  for (int32_t i = r - 1; i >= 0; --i) {
    double s = qtb[i];
    for (int32_t j = i + 1; j < r; ++j) s -= W[(int64_t)i * p + j] * y[j];
    y[i] = s / W[(int64_t)i * p + i];
  }
  /* z = Z^T [y; 0]: apply reflectors in reverse application order */
  for (int32_t i = 0; i < r; ++i) {
    if (ztau[i] == 0.0) continue;
    const double* v = zv + (int64_t)i * p;
    double s = y[i];
    for (int32_t j = r; j < p; ++j) s += v[j] * y[j];
    s *= ztau[i];
    y[i] -= s;
    for (int32_t j = r; j < p; ++j) y[j] -= s * v[j];
  }
  for (int32_t j = 0; j < p; ++j) x[perm[j]] = y[j];
  free(W);
  free(zv);
  free(ztau);
  free(y);
}

/* direct_lingam.cpp:46-70 — centred (not standardised) data; per target p, regress
 * X[:, order[p]] on X[:, order[0..p-1]]. */
/* Targets at the listed order positions only (positions == NULL: every p >= 1). */
static int fit_weights_impl(const double* X, int64_t n, int32_t d, int64_t ld, const int32_t* order,
                            const int32_t* positions, int32_t npos, double* B, int32_t* used_pinv, orc_status* st) {
  double* centered = (double*)malloc(sizeof(double) * (size_t)n * (size_t)d);
  for (int32_t j = 0; j < d; ++j) {
    const double* c = X + (int64_t)j * ld;
    const double m = orc_mean(c, n); /* Eigen colwise().mean(): plain sum / n */
    for (int64_t i = 0; i < n; ++i) centered[i + n * j] = c[i] - m;
  }
  memset(B, 0, sizeof(double) * (size_t)d * (size_t)d);
  *used_pinv = 0;
  double* A = (double*)malloc(sizeof(double) * (size_t)n * (size_t)(d > 1 ? d - 1 : 1));
  double* b = (double*)malloc(sizeof(double) * (size_t)n);
  double* hcoef = (double*)malloc(sizeof(double) * (size_t)d);
  int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)d);
  double* coef = (double*)malloc(sizeof(double) * (size_t)d);
  const int32_t count = positions ? npos : (d > 1 ? d - 1 : 0);
  for (int32_t e = 0; e < count; ++e) {
    const int32_t p = positions ? positions[e] : e + 1;
    if (p < 1 || p >= d) continue;
    const int32_t target = order[p];
    for (int32_t q = 0; q < p; ++q)
      memcpy(A + n * q, centered + n * order[q], sizeof(double) * (size_t)n);
    memcpy(b, centered + n * target, sizeof(double) * (size_t)n);
    const int32_t rank = colpiv_qr(A, n, p, hcoef, perm);
    const int32_t kk = (int32_t)(n < p ? n : p);
    apply_qt(A, n, kk, hcoef, b);
    if (rank < p) {
      cod_solve(A, n, p, rank, perm, b, coef);
      *used_pinv = 1;
    } else {
      double* y = (double*)malloc(sizeof(double) * (size_t)p);
      for (int32_t i = p - 1; i >= 0; --i) {
        double s = b[i];
        for (int32_t j = i + 1; j < p; ++j) s -= A[i + n * j] * y[j];
        y[i] = s / A[i + n * i];
      }
      for (int32_t j = 0; j < p; ++j) coef[perm[j]] = y[j];
      free(y);
    }
    for (int32_t q = 0; q < p; ++q) B[target + (int64_t)d * order[q]] = coef[q];
  }
  free(centered);
  free(A);
  free(b);
  free(hcoef);
  free(perm);
  free(coef);
  return ok(st);
}

/* direct_lingam.cpp:46-70 — centred (not standardised) data; per target p, regress
 * X[:, order[p]] on X[:, order[0..p-1]]. */
int orc_fit_weights(const double* X, int64_t n, int32_t d, int64_t ld, const int32_t* order,
                    double* B, int32_t* used_pinv, orc_status* st) {
  return fit_weights_impl(X, n, d, ld, order, NULL, 0, B, used_pinv, st);
}

int orc_fit_weights_targets(const double* X, int64_t n, int32_t d, int64_t ld, const int32_t* order,
                            const int32_t* positions, int32_t npos, double* B, int32_t* used_pinv, orc_status* st) {
  return fit_weights_impl(X, n, d, ld, order, positions, npos, B, used_pinv, st);
}

/* ------------------------------------------------- weights: one prefix QR for all targets
 *
 * The same least-squares problems as orc_fit_weights (direct_lingam.cpp:46-70), from ONE
 * Householder QR of the order-permuted centred design A = [x_o0 - m, ..., x_o(d-1) - m]:
 * the predecessor design of target p is A's first p columns, so the QR of A restricted
 * to them gives target p's regression (coordinates of column p in the first rows, solved
 * against the leading triangle). Rank deficiency is handled in echelon form: a column
 * whose residual norm (after the reflectors of the columns before it) is at or below the
 * ColPivHouseholderQR threshold of the first design it enters, eps * min(n, k + 1) *
 * max_{j <= k} ||a_j|| (Eigen's rank(): |R_ii| > |max pivot| * eps * diagonalSize, the max
 * pivot being the largest column norm), gets no reflector: it is "dependent", A_S = Q_r T
 * with T r x p echelon. For target p with independent predecessors I and dependent ones D:
 *   a  = T_I^-1 c   (c: column p's first r coordinates)      -- every LS solution has
 *   b_I = a - G b_D (G: columns g_k = T_I^-1 T[:, k], k in D)  -- this form, and the
 *   b_D = (I + G^T G)^-1 G^T a                                 -- minimum-norm one
 * which is what CompleteOrthogonalDecomposition::solve returns (direct_lingam.cpp:62).
 * Full-rank targets reduce to the plain QR solution (direct_lingam.cpp:64). */

typedef struct {
  double* A;        /* n x d, column-major (lda = n), factorised in place */
  int64_t n;
  int32_t d;
  int32_t nthreads;
  int32_t tid;
  pthread_barrier_t* bar;
  /* shared per-step state */
  volatile int32_t* step_row; /* row of the current reflector, -1 when the column is dependent */
  volatile double* step_tau;
} pqr_job;

static void* pqr_worker(void* arg) {
  pqr_job* J = (pqr_job*)arg;
  const int64_t n = J->n;
  for (int32_t k = 0; k < J->d; ++k) {
    pthread_barrier_wait(J->bar); /* thread 0 has built reflector k (or marked it dependent) */
    const int32_t r = J->step_row[k];
    if (r >= 0) {
      const double tau = J->step_tau[k];
      const double* v = J->A + n * k;
      for (int32_t j = k + 1 + J->tid; j < J->d; j += J->nthreads) {
        double* cj = J->A + n * j;
        double s = cj[r];
        for (int64_t i = r + 1; i < n; ++i) s += v[i] * cj[i];
        s *= tau;
        cj[r] -= s;
        for (int64_t i = r + 1; i < n; ++i) cj[i] -= s * v[i];
      }
    }
    pthread_barrier_wait(J->bar); /* column k + 1 is up to date */
  }
  return NULL;
}

/* Cholesky solve of the small SPD system N x = y (N m x m row-major, overwritten). */
static void spd_solve(double* N, int32_t m, double* y) {
  for (int32_t j = 0; j < m; ++j) {
    double s = N[(int64_t)j * m + j];
    for (int32_t k = 0; k < j; ++k) s -= N[(int64_t)j * m + k] * N[(int64_t)j * m + k];
    const double l = sqrt(s);
    N[(int64_t)j * m + j] = l;
    for (int32_t i = j + 1; i < m; ++i) {
      double t = N[(int64_t)i * m + j];
      for (int32_t k = 0; k < j; ++k) t -= N[(int64_t)i * m + k] * N[(int64_t)j * m + k];
      N[(int64_t)i * m + j] = t / l;
    }
  }
  for (int32_t i = 0; i < m; ++i) {
    double t = y[i];
    for (int32_t k = 0; k < i; ++k) t -= N[(int64_t)i * m + k] * y[k];
    y[i] = t / N[(int64_t)i * m + i];
  }
  for (int32_t i = m - 1; i >= 0; --i) {
    double t = y[i];
    for (int32_t k = i + 1; k < m; ++k) t -= N[(int64_t)k * m + i] * y[k];
    y[i] = t / N[(int64_t)i * m + i];
  }
}

typedef struct {
  const double* A;
  int64_t n;
  int32_t d;
  const int32_t* rbefore; /* rows (reflectors) before column k */
  const int32_t* rowcol;  /* column of reflector t */
  const int32_t* dep;     /* dependent columns, ascending */
  int32_t ndep;
  double* coef;           /* d x d: row k = a_k (length rbefore[k]) */
  int32_t tid, nthreads;
} pqr_solve_job;

/* a_k = T_I^-1 c_k for every column k (targets, and g_k for dependent columns). */
static void* pqr_solve_worker(void* arg) {
  pqr_solve_job* J = (pqr_solve_job*)arg;
  const int64_t n = J->n;
  for (int32_t k = J->tid; k < J->d; k += J->nthreads) {
    const int32_t r = J->rbefore[k];
    double* a = J->coef + (int64_t)k * J->d;
    for (int32_t i = 0; i < r; ++i) a[i] = J->A[i + n * k];
    for (int32_t t = r - 1; t >= 0; --t) {
      const double* col = J->A + n * J->rowcol[t];
      a[t] /= col[t];
      for (int32_t i = 0; i < t; ++i) a[i] -= a[t] * col[i];
    }
  }
  return NULL;
}

int orc_fit_weights_prefix(const double* X, int64_t n, int32_t d, int64_t ld, const int32_t* order,
                           int32_t nthreads, double* B, int32_t* used_pinv, int32_t* n_dependent,
                           orc_status* st) {
  if (nthreads < 1) nthreads = 1;
  memset(B, 0, sizeof(double) * (size_t)d * (size_t)d);
  *used_pinv = 0;
  if (n_dependent) *n_dependent = 0;
  if (d < 2) return ok(st);
  double* A = (double*)malloc(sizeof(double) * (size_t)n * (size_t)d);
  double* cn = (double*)malloc(sizeof(double) * (size_t)d);
  for (int32_t k = 0; k < d; ++k) {
    const double* c = X + (int64_t)order[k] * ld;
    const double m = orc_mean(c, n); /* Eigen colwise().mean() (direct_lingam.cpp:49) */
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      A[i + n * k] = c[i] - m;
      s += A[i + n * k] * A[i + n * k];
    }
    cn[k] = sqrt(s);
  }
  int32_t* step_row = (int32_t*)malloc(sizeof(int32_t) * (size_t)d);
  double* step_tau = (double*)malloc(sizeof(double) * (size_t)d);
  int32_t* rbefore = (int32_t*)malloc(sizeof(int32_t) * (size_t)d);
  int32_t* rowcol = (int32_t*)malloc(sizeof(int32_t) * (size_t)d);
  int32_t* dep = (int32_t*)malloc(sizeof(int32_t) * (size_t)d);
  int32_t ndep = 0;

  pthread_barrier_t bar;
  pthread_barrier_init(&bar, NULL, (unsigned)nthreads);
  pqr_job* jobs = (pqr_job*)calloc((size_t)nthreads, sizeof(pqr_job));
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int32_t t = 0; t < nthreads; ++t) {
    jobs[t] = (pqr_job){A, n, d, nthreads, t, &bar, step_row, step_tau};
    if (t) pthread_create(&th[t], NULL, pqr_worker, &jobs[t]);
  }
  /* thread 0 = this thread: builds reflector k, then shares the update of columns > k */
  int32_t r = 0;
  double maxnorm = 0.0;
  for (int32_t k = 0; k < d; ++k) {
    if (cn[k] > maxnorm) maxnorm = cn[k];
    const double thr = 2.220446049250313e-16 * (double)((int64_t)(k + 1) < n ? (k + 1) : n) * maxnorm;
    double* col = A + n * k;
    rbefore[k] = r;
    double tail = 0.0;
    for (int64_t i = r + 1; i < n; ++i) tail += col[i] * col[i];
    const double c0 = r < n ? col[r] : 0.0;
    const double nu = sqrt(c0 * c0 + tail);
    if (r < n && nu > thr) {
      double beta = c0 >= 0.0 ? -nu : nu, tau;
      if (tail == 0.0) {
        tau = 0.0;
        beta = c0;
      } else {
        const double denom = c0 - beta;
        for (int64_t i = r + 1; i < n; ++i) col[i] /= denom;
        tau = (beta - c0) / beta;
      }
      col[r] = beta;
      step_row[k] = r;
      step_tau[k] = tau;
      rowcol[r] = k;
      ++r;
    } else {
      step_row[k] = -1;
      dep[ndep++] = k;
    }
    pthread_barrier_wait(&bar);
    {
      const int32_t rr = step_row[k];
      if (rr >= 0) {
        const double tau = step_tau[k];
        for (int32_t j = k + 1; j < d; j += nthreads) {
          double* cj = A + n * j;
          double s = cj[rr];
          for (int64_t i = rr + 1; i < n; ++i) s += col[i] * cj[i];
          s *= tau;
          cj[rr] -= s;
          for (int64_t i = rr + 1; i < n; ++i) cj[i] -= s * col[i];
        }
      }
    }
    pthread_barrier_wait(&bar);
  }
  for (int32_t t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  pthread_barrier_destroy(&bar);

  /* every column's coordinates solved against the leading triangle */
  double* coef = (double*)calloc((size_t)d * (size_t)d, sizeof(double));
  pqr_solve_job* sj = (pqr_solve_job*)calloc((size_t)nthreads, sizeof(pqr_solve_job));
  for (int32_t t = 0; t < nthreads; ++t) {
    sj[t] = (pqr_solve_job){A, n, d, rbefore, rowcol, dep, ndep, coef, t, nthreads};
    if (t) pthread_create(&th[t], NULL, pqr_solve_worker, &sj[t]);
  }
  pqr_solve_worker(&sj[0]);
  for (int32_t t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);

  double* bD = (double*)malloc(sizeof(double) * (size_t)(ndep > 0 ? ndep : 1));
  double* N = (double*)malloc(sizeof(double) * (size_t)(ndep > 0 ? ndep : 1) * (size_t)(ndep > 0 ? ndep : 1));
  double* bI = (double*)malloc(sizeof(double) * (size_t)d);
  for (int32_t p = 1; p < d; ++p) {
    const int32_t target = order[p];
    const int32_t rp = rbefore[p];
    const double* a = coef + (int64_t)p * d;
    int32_t m = 0;
    while (m < ndep && dep[m] < p) ++m; /* dependent predecessors dep[0..m) */
    for (int32_t t = 0; t < rp; ++t) bI[t] = a[t];
    if (m > 0) {
      *used_pinv = 1;
      /* N = I + G^T G, y = G^T a (g_k zero beyond rbefore[k]) */
      for (int32_t i = 0; i < m; ++i) {
        const double* gi = coef + (int64_t)dep[i] * d;
        const int32_t ri = rbefore[dep[i]];
        double s = 0.0;
        for (int32_t t = 0; t < ri; ++t) s += gi[t] * a[t];
        bD[i] = s;
        for (int32_t j = 0; j <= i; ++j) {
          const double* gj = coef + (int64_t)dep[j] * d;
          const int32_t rj = rbefore[dep[j]];
          const int32_t rm = ri < rj ? ri : rj;
          double g = 0.0;
          for (int32_t t = 0; t < rm; ++t) g += gi[t] * gj[t];
          N[(int64_t)i * m + j] = N[(int64_t)j * m + i] = g + (i == j ? 1.0 : 0.0);
        }
      }
      spd_solve(N, m, bD);
      for (int32_t i = 0; i < m; ++i) {
        const double* gi = coef + (int64_t)dep[i] * d;
        const int32_t ri = rbefore[dep[i]];
        for (int32_t t = 0; t < ri; ++t) bI[t] -= gi[t] * bD[i];
        B[target + (int64_t)d * order[dep[i]]] = bD[i];
      }
    }
    for (int32_t t = 0; t < rp; ++t) B[target + (int64_t)d * order[rowcol[t]]] = bI[t];
  }
  if (n_dependent) *n_dependent = ndep;
  free(bD);
  free(N);
  free(bI);
  free(coef);
  free(sj);
  free(jobs);
  free(th);
  free(A);
  free(cn);
  free(step_row);
  free(step_tau);
  free(rbefore);
  free(rowcol);
  free(dep);
  return ok(st);
}
