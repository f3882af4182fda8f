/*
 * plingam_b200.h — C-ABI of the B200 DirectLiNGAM causal-order engine
 * (libplingam_b200.so). Plain pointers and sizes; no exceptions cross this boundary;
 * the caller owns every buffer, the library copies inputs and never retains pointers.
 *
 * Each entry point replaces one reference interface (paths relative to
 * /root/reference/proj); see INTEGRATION.md for the bindings a maintainer would add.
 *
 * Matrices are column-major FP64 (each variable contiguous), n samples x d variables,
 * leading dimension ld >= n — the layout of plingam::DataMatrix (include/plingam/types.hpp:14-30).
 *
 * Status: code 0 = ok, otherwise 1 + ordinal of plingam::ErrorCode
 * (include/plingam/error.hpp:10-27); row/col carry the reference's Error::row()/col()
 * (-1 when not meaningful). Every function returns st->code.
 */
#ifndef PLINGAM_B200_H
#define PLINGAM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct plg_status {
  int32_t code;
  int64_t row;
  int64_t col;
  char msg[256];
} plg_status;

enum plg_error_code {
  PLG_OK = 0,
  PLG_NonFinite = 1,
  PLG_ZeroVariance = 2,
  PLG_TooFewSamples = 3,
  PLG_TooShort = 4,
  PLG_LengthMismatch = 5,
  PLG_DimensionMismatch = 6,
  PLG_EmptyCandidates = 7,
  PLG_SingularDesign = 8,
  PLG_InsufficientRows = 9,
  PLG_UnstableSystem = 10,
  PLG_OutOfRange = 11,
  PLG_InvalidIndex = 12,
  PLG_CudaError = 100, /* device/runtime failure (no reference counterpart) */
  PLG_NcclError = 101
};

/* Per-call measurements of the last causal_order / search on this context. */
typedef struct plg_stats {
  double total_ms;      /* device time of the whole call (CUDA events on the engine stream) */
  double pair_ms;       /* device time of the pair-evaluation launches (exhaustive rounds: pair
                           kernel + finalize; pruned rounds: the pair-list kernel) */
  double h2d_ms;        /* host->device copy of X (host entry points only) */
  int64_t pair_evals;   /* ordered (i, j) pair evaluations of the reference's Alg. 1 */
  int64_t ede;          /* element-direction evaluations (= n * pair_evals) */
  int64_t pairs_evaluated; /* unordered pairs whose two residual entropies were actually
                              computed (exact pruning skips pairs that cannot change the order) */
  int64_t launches;     /* kernels launched by the call */
  int64_t pair_launches; /* pair-evaluation launches timed into pair_ms */
  int32_t rounds;
  int32_t world;
  int64_t h2d_bytes;
  int64_t d2h_bytes;
  double resid_ms;      /* device time of the residualisation launches (fused with the next
                           round's column entropies) */
  int64_t resid_bytes;  /* their algorithmic HBM bytes: (2 (u - 1) + 1) n 8 per round */
  /* Near-tie guard (causal_order): rounds whose runner-up k is not certified above
   * winner k * (1 + 1e-9) — the reference's strict '>' argmax (ordering.cpp:154-160) could
   * pick differently there under its own rounding — and the smallest relative gap
   * (runner-up k - winner k) / winner k over all rounds, with its round. */
  int32_t near_ties;
  int32_t min_gap_round;
  double min_gap;
} plg_stats;

typedef struct plg_ctx plg_ctx;

/* Library version string, e.g. "plingam_b200 0.1.0 (sm_100a)". */
const char* plg_version(void);

/* One engine on one device (replaces the CPU worker pool of ordering.cpp:114-146). */
int plg_ctx_create(int32_t device, plg_ctx** out, plg_status* st);

/* Multi-GPU: one process per GPU. Every rank passes the same 128-byte NCCL unique id
 * (from plg_nccl_unique_id on rank 0). The data are replicated; rank r evaluates its
 * contiguous share of the pair tiles and one ncclAllGather per round exchanges the
 * entropies, so every rank holds the identical order. */
int plg_nccl_unique_id(void* out_128_bytes, plg_status* st);
int plg_ctx_create_dist(int32_t device, int32_t rank, int32_t world, const void* nccl_uid_128,
                        plg_ctx** out, plg_status* st);

/* Multi-GPU through peer memory (no collective library): one process per GPU. Each rank
 * creates its context with the same world size and max_dims (largest d it will be called
 * with: sizes the exchange arena, 2 x (d^2 + d) + 2 x round-0 tile table doubles), exports the
 * 64-byte CUDA IPC handle of its arena with plg_p2p_handle, the caller gathers the handles of
 * all ranks in rank order (any host channel: torch.distributed, MPI, a file) and every rank
 * calls plg_p2p_connect with the world x 64 bytes. Every exchange is then a store of each
 * produced value into every rank's arena (NVLink) plus a device-side flag barrier: no host
 * synchronisation inside a call. world = 1 runs every exchange through its own arena (a
 * self-test of the exchange path). Calls must be made collectively by all ranks with the
 * same inputs, as for plg_ctx_create_dist. At most 8 ranks. */
int plg_ctx_create_p2p(int32_t device, int32_t rank, int32_t world, int32_t max_dims, plg_ctx** out,
                       plg_status* st);
int plg_p2p_handle(plg_ctx* ctx, void* out_64_bytes, plg_status* st);
int plg_p2p_connect(plg_ctx* ctx, const void* handles_world_x_64_bytes, plg_status* st);
void plg_ctx_destroy(plg_ctx* ctx);

/* plingam::causal_order(X, parallel, workers) — ordering.hpp:42, ordering.cpp:213-244.
 * X in host memory; order_out: d ints. */
int plg_causal_order(plg_ctx* ctx, const double* X, int64_t n, int32_t d, int64_t ld,
                     int32_t* order_out, plg_status* st);

/* Same, with X already resident in device memory of ctx's device. */
int plg_causal_order_device(plg_ctx* ctx, const double* dX, int64_t n, int32_t d, int64_t ld,
                            int32_t* order_out, plg_status* st);

/* Exact pruning of causal_order's search rounds (default on; environment PLG_PRUNE=0 turns
 * it off at context creation). A pruned round evaluates only the pairs needed to prove its
 * argmin: rows whose partial k (a sum over a subset of non-negative terms) already exceeds
 * an exactly computed k cannot win. The order is identical to the exhaustive rounds' and
 * the winner's k has the same bits; only non-winning scores are left uncomputed, which
 * causal_order never returns. plg_search always evaluates every pair. */
int plg_set_prune(plg_ctx* ctx, int32_t enable, plg_status* st);
/* The winning k (= -score of the chosen variable) of every round of the last causal_order on
 * ctx, in round order (count = min(cap, rounds)). Diagnostics and parity tests. */
int plg_last_round_k(plg_ctx* ctx, double* out, int32_t cap, int32_t* count, plg_status* st);
/* Per round of the last causal_order: a lower bound of the runner-up's k (exact when the
 * runner-up row was fully evaluated — every row within k* (1 + 1e-9) is — else that row's
 * partial k), so second - k (plg_last_round_k) bounds the best-vs-second gap from below. */
int plg_last_round_gaps(plg_ctx* ctx, double* second_out, int32_t cap, int32_t* count, plg_status* st);
/* plingam::search_causal_order(X, U) — ordering.hpp:27, ordering.cpp:101-168.
 * scores_out: d doubles, -inf for non-candidates, -k for candidates. */
int plg_search(plg_ctx* ctx, const double* X, int64_t n, int32_t d, int64_t ld, const int32_t* U,
               int32_t u, int32_t* chosen_out, double* scores_out, plg_status* st);

/* plingam::regress_out(X, exog, remaining) — ordering.hpp:38, ordering.cpp:178-211.
 * out: n x r column-major (ld = n). */
int plg_regress_out(plg_ctx* ctx, const double* X, int64_t n, int32_t d, int64_t ld, int32_t exog,
                    const int32_t* remaining, int32_t r, double* out, plg_status* st);

/* Adjacency weights of DirectLingam::fit (direct_lingam.cpp:46-70) given an order:
 * B (d x d, column-major, B[target + d * pred]). Every predecessor regression at once from
 * one FP64 Householder QR of the order-permuted centred design, in echelon form: a column
 * whose residual norm is at or below ColPivHouseholderQR's rank threshold
 * (eps * min(n, p) * largest column norm, direct_lingam.cpp:57-59) gets no reflector, and
 * the targets after it take the minimum-norm least-squares solution, as
 * CompleteOrthogonalDecomposition (direct_lingam.cpp:60-63); used_pinv is then set.
 * Entirely on the device. */
int plg_fit_weights(plg_ctx* ctx, const double* X, int64_t n, int32_t d, int64_t ld,
                    const int32_t* order, double* B_out, int32_t* used_pinv, plg_status* st);

/* VarLiNGAM front-end (var_lingam.cpp:7-53, estimate_var): least-squares VAR(lag) with
 * intercept of the T x d series ts. coef_out (optional): (1 + lag d) x d column-major, row 0
 * the intercepts, row 1 + (tau - 1) d + j the coefficient of x_j(t - tau); resid_out
 * (optional): (T - lag) x d residuals. Device: scaled normal equations, blocked Cholesky,
 * one refinement step. Errors: OutOfRange (lag < 1), DimensionMismatch, NonFinite,
 * InsufficientRows (T < lag + 2d or fewer rows than coefficients), SingularDesign. */
int plg_estimate_var(plg_ctx* ctx, const double* ts, int64_t T, int32_t d, int64_t ld, int32_t lag,
                     double* coef_out, double* resid_out, plg_status* st);
/* VarLiNGAM lag weights (var_lingam.cpp:55-70): out[t] = (I - B0) M[t] for t < lag, all d x d
 * column-major (M and out hold lag matrices back to back). */
int plg_var_lagged_weights(plg_ctx* ctx, const double* B0, const double* M, int32_t d, int32_t lag, double* out,
                           plg_status* st);
/* The element functions of plingam::kernels (include/plingam/kernels.hpp:25-70), exposed
 * by the reference's Python module (bindings/pymodule.cpp:79-96):
 *   standardize (kernels.cpp:92-104; bit-identical: left-to-right sums),
 *   residual (kernels.cpp:106-121; bit-identical), entropy_approx (:123-132),
 *   entropy_of_normalized (:134-148), diff_mutual_info (:150-159; exactly antisymmetric).
 * Entropies use the engine's table-driven FP64 element math (a few ulp from libm). */
int plg_standardize(plg_ctx* ctx, const double* x, int64_t n, double* out, plg_status* st);
int plg_residual(plg_ctx* ctx, const double* xi, int64_t ni, const double* xj, int64_t nj, double* out,
                 plg_status* st);
int plg_entropy_approx(plg_ctx* ctx, const double* u, int64_t n, double* out, plg_status* st);
int plg_entropy_of_normalized(plg_ctx* ctx, const double* r, int64_t n, double* out, plg_status* st);
int plg_diff_mutual_info(plg_ctx* ctx, const double* xi_std, const double* xj_std, const double* ri_j,
                         const double* rj_i, int64_t n, double* out, plg_status* st);

/* Round schedule (host-only, no device needed): the rank's contiguous share of the pair
 * tiles and the round's sample segmentation. The segmentation depends only on (u, n), so
 * every pair entropy has the same bits for any world size. */
typedef struct plg_round_plan {
  int32_t nb;             /* 32-wide position blocks: ceil(u / 32) */
  int32_t ntiles;         /* upper-triangle tiles nb (nb + 1) / 2 */
  int32_t tiles_per_rank; /* ceil(ntiles / world); rank r owns [r * tpr, min(ntiles, (r+1) * tpr)) */
  int32_t tile_begin;
  int32_t tile_count;
  int32_t nseg;
  int32_t seg_len;
  int32_t replicated;     /* u <= 128: every rank evaluates every pair (tile_begin 0, tile_count
                             ntiles) and the round has no exchange; the segmentation is then
                             that of the compact small-round kernel */
} plg_round_plan;
int plg_plan_round(int32_t u, int64_t n, int32_t rank, int32_t world, plg_round_plan* out);
/* Pruned rounds across ranks (host-only): each stage's pair list (identical on every rank)
 * is split into contiguous slices; rank r evaluates entries [begin, end) and contributes a
 * slot of `slot` entries (= ceil(total / world)) to the stage's in-place all-gather of M. */
int plg_plan_list_shard(int32_t total, int32_t rank, int32_t world, int32_t* begin, int32_t* end,
                        int32_t* slot);
/* tile index -> (bi, bj), bi <= bj, row-major over the upper triangle */
int plg_tile_decode(int32_t t, int32_t nb, int32_t* bi, int32_t* bj);

/* Per-launch timing of the pair-evaluation and residualisation launches (plg_stats.pair_ms,
 * resid_ms; default off). Off: only the call's total device time is measured, which saves
 * the host ~10k event queries per large causal order. */
int plg_set_detail_timing(plg_ctx* ctx, int32_t enable, plg_status* st);
/* Stats of the last call on ctx. */
int plg_last_stats(plg_ctx* ctx, plg_stats* out);

/* Sampled-round state: run the first `rounds` rounds of causal_order and
 * return the working state the next round would search: the active variables (ascending)
 * and their current working columns (n x u_active, column-major). Scale-equivalent to
 * the reference's `working` matrix columns (standardisation absorbs the scale). */
int plg_round_state(plg_ctx* ctx, const double* X, int64_t n, int32_t d, int64_t ld,
                    int32_t rounds, int32_t* active_out, int32_t* n_active, double* cols_out,
                    int32_t* order_prefix_out, plg_status* st);

/* Analysis hook (not part of the reference surface): when set, causal_order on a
 * single-rank context synchronises after every round's k reduction and calls
 * hook(user, round, u, active (u ints, position -> variable), E (u*u doubles,
 * E[p*u+q] = E(p|q)), H (u), k (u)). Pass NULL to clear. */
typedef void (*plg_round_hook)(void* user, int32_t round, int32_t u, const int32_t* active,
                               const double* E, const double* H, const double* k);
int plg_debug_set_round_hook(plg_ctx* ctx, plg_round_hook hook, void* user);
/* Test hook: element functions on device for a host vector u (n values): out[4i..4i+3] =
 * {log cosh (table path), u e^{-u^2/2} (table path), libdevice log cosh, libdevice pdf}. */
int plg_math_probe(plg_ctx* ctx, const double* u, int64_t n, double* out, plg_status* st);

#ifdef __cplusplus
}
#endif
#endif
