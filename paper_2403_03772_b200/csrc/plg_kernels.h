// plg_kernels.h — launchers for the sm_100a kernels of the causal-order engine.
// Internal to libplingam_b200.so (the C-ABI in include/plingam_b200.h is the boundary).
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>

namespace plg {

// Per-device once-values. Kernel attributes (the dynamic shared memory opt-in above 48 KB)
// and occupancy-derived grids belong to the device current at launch, so a process that
// switches devices (set_device, one context per GPU) must not reuse another device's.
constexpr int kMaxDevices = 64;
struct DeviceCache {
  std::atomic<int> v[kMaxDevices] = {};
  template <class F>
  int get(F f) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::atomic<int>& a = v[dev & (kMaxDevices - 1)];
    int x = a.load(std::memory_order_acquire);
    if (!x) {
      x = f();
      a.store(x, std::memory_order_release);
    }
    return x;
  }
};

constexpr int kBT = 32;           // active positions per tile side
constexpr int kTilePairs = kBT * kBT;
constexpr int kCH = 64;           // samples per shared-memory stage
constexpr int kCHS = kCH + 2;     // padded column stride in shared memory (doubles)
constexpr int kSegMin = 256;      // smallest sample segment per CTA

// Error key: first error in the reference's raising order (ordering.cpp build_cache
// before candidate_score, rounds ascending). key = round<<40 | kind<<32 | (col+1).
constexpr unsigned long long kNoError = ~0ull;
enum ErrKind : unsigned { kErrColZeroVar = 0, kErrPairCollinear = 1, kErrInternal = 255 };

__host__ __device__ inline unsigned long long err_key(int round, unsigned kind, int col) {
  return (static_cast<unsigned long long>(round) << 40) |
         (static_cast<unsigned long long>(kind) << 32) | static_cast<unsigned>(col + 1);
}

struct RoundState {  // device-resident per-round scalars
  int chosen_pos;
  int chosen_col;
};

// Column-major tile upper triangle: tile index -> (bi, bj), bi <= bj.
__host__ __device__ inline void tile_decode(int t, int nb, int& bi, int& bj) {
  int row = 0, start = 0;
  while (t >= start + (nb - row)) {
    start += nb - row;
    ++row;
  }
  bi = row;
  bj = row + (t - start);
}

// ---- peer-memory exchange (multi-rank contexts created with plg_ctx_create_p2p) ----
// Every rank owns one exchange arena; all ranks map every arena (CUDA IPC over NVLink). A
// kernel that produces exchanged values stores each one into its local arena position and
// the same offset of every peer's arena (peer_store), then a signal kernel publishes a
// sequence number into every peer's flag slot for this rank and the consumer's wait kernel
// waits for every rank's slot (p2p_kernels.cu). No host synchronisation, no collective.
constexpr int kMaxPeers = 8;
struct PeerTable {
  int n = 0;  // ranks mirrored to (0: local only, no exchange through peer memory)
  int rank = 0;
  char* base[kMaxPeers] = {};  // every rank's arena as mapped in this process (base[rank]: own)
};
// Arena layout (byte offsets): flags [0, 1024): u64 {signals sent, unused, peer r's last
// signal at 2 + r}; errs (two parities x kMaxPeers u64) at 1024; then pres[2] and epack[2].
constexpr int64_t kArenaFlags = 0;
constexpr int64_t kArenaErrs = 1024;
constexpr int64_t kArenaData = 2048;
#ifdef __CUDACC__
__device__ __forceinline__ void peer_store(const PeerTable& pt, double* local, double v) {
  const int64_t off = reinterpret_cast<char*>(local) - pt.base[pt.rank];
#pragma unroll 1
  for (int r = 0; r < pt.n; ++r) *reinterpret_cast<double*>(pt.base[r] + off) = v;
}
// One thread: publish this rank's next sequence number in every rank's flag slot for it
// (after the caller's stores; release at system scope). Returns the sequence number.
__device__ __forceinline__ unsigned long long p2p_signal_dev(const PeerTable& pt) {
  unsigned long long* f = reinterpret_cast<unsigned long long*>(pt.base[pt.rank] + kArenaFlags);
  const unsigned long long seq = f[0] + 1;
  f[0] = seq;
  __threadfence_system();
#pragma unroll 1
  for (int r = 0; r < pt.n; ++r) {
    unsigned long long* slot = reinterpret_cast<unsigned long long*>(pt.base[r] + kArenaFlags) + 2 + pt.rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(slot), "l"(seq) : "memory");
  }
  return seq;
}
// One thread: until every rank has signalled as often as this rank (every rank signals once
// per exchange, so this rank's count is the exchange's sequence number).
__device__ __forceinline__ void p2p_wait_dev(const PeerTable& pt) {
  const unsigned long long* f = reinterpret_cast<const unsigned long long*>(pt.base[pt.rank] + kArenaFlags);
  const unsigned long long target = *reinterpret_cast<const volatile unsigned long long*>(f);
#pragma unroll 1
  for (int r = 0; r < pt.n; ++r) {
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f + 2 + r) : "memory");
      if (v >= target) break;
      __nanosleep(200);
    }
  }
}
#endif
// signal: this rank's error key into every peer's errs[parity][rank] (err_off >= 0), a
// system-scope fence, then the next sequence number into every peer's flag slot for this rank
void launch_p2p_signal(const PeerTable& pt, const unsigned long long* err, int64_t err_off, cudaStream_t s);
// wait: until every rank's flag slot in the local arena holds this rank's next expected sequence
void launch_p2p_wait(const PeerTable& pt, cudaStream_t s);

struct PairLaunch {
  const double* W;
  int64_t ldw;
  int64_t n;
  const double* C;
  int64_t ldc;
  const int* act;
  int u;
  int nb;
  int tile_begin;  // global tile index of this launch's first tile
  int ntiles;      // tiles in this launch
  int seg_len;
  int nseg;
  double* part;    // [ntiles][nseg][kTilePairs][4]
  double* epack;   // [global tiles][2][kBT][kBT]
  const double* g_exp;
  const double2* g_log;
  unsigned long long* err;
  int round;
  PeerTable peers;  // n > 0: the entropy tiles are also stored into every rank's epack (same offset)
};

void launch_pair(const PairLaunch& a, cudaStream_t s);
void launch_finalize(const PairLaunch& a, cudaStream_t s);

// Small active sets (u <= kSmallU): one thread per unordered pair (p < q, p-major) and
// sample segment, columns read through L1 (the u columns sit in L2). Computed on every rank
// (no exchange); part = [nseg][npairs][4]; the finalize writes the same epack layout.
constexpr int kSmallU = 128;
constexpr int kSmallThreads = 256;
void launch_pair_small(const PairLaunch& a, cudaStream_t s);
void launch_finalize_small(const PairLaunch& a, cudaStream_t s);

// H[p] = entropy(w_col / sqrt(C_col,col)) for active positions p < u. For round > 0 it
// is also build_cache's ZeroVariance(col) check (ordering.cpp:56-62): a column whose
// residualisation left it identically zero (nz[col] != round) or whose partial variance
// is not positive.
void launch_colent(const double* W, int64_t ldw, int64_t n, const double* C, int64_t ldc,
                   const int* act, int u, double* H, const double* g_exp, const double2* g_log,
                   const int* nz, const int* col_var, int round, unsigned long long* err,
                   cudaStream_t s);

// In-place residualisation w_r <- w_r - (C_rm / C_mm) w_m (multiply then subtract, as
// residual_into, kernels.cpp:81-85; nz[r] = tag when the new column has a nonzero entry)
// fused with the next round's column-entropy sums per
// chunk of kResidChunk samples (hpart: [ur][resid_chunks(n)][2]); launch_hfin turns them into
// H (and runs colent's zero-variance check). Rounds >= 1 of causal_order use this pair.
constexpr int64_t kResidChunk = 1024;
int resid_chunks(int64_t n);
// C_updated: C already holds the updated Gram (in-place update before this launch); else C is
// the pre-update Gram and each column's new C_rr is recomputed (gram_update_entry).
void launch_resid_ent(double* W, int64_t ldw, int64_t n, const double* C, int64_t ldc, const int* act_nxt, int ur,
                      const RoundState* rs, int* nz, int tag, const unsigned long long* err, double* hpart,
                      const double* g_exp, const double2* g_log, cudaStream_t s, bool C_updated = true);
void launch_hfin(const double* hpart, int64_t n, const double* C, int64_t ldc, const int* act, int u, double* H,
                 const int* nz, const int* col_var, int round, unsigned long long* err, cudaStream_t s);

// Validation + round-0 standardisation with the reference's left-to-right sums
// (types.cpp:21-47, kernels.cpp:44-57,92-104). col_map[c] = source column of local c.
// stat[c] = {first non-finite row or -1, zero-variance flag}.
// msd (optional): {mean, sd} per column.
void launch_standardize(const double* X, int64_t ldx, int64_t n, const int* col_map, int ncol,
                        double* W, int64_t ldw, int* stat, double* msd, int check_finite,
                        cudaStream_t s);

// C = W^T W / n (FP64, symmetric, deterministic order). Few 64x64 output tiles (small d)
// split the sample axis into chunks reduced in ascending order through `scratch`
// (gram_scratch_doubles(ncol, n) doubles); the split is a pure function of (ncol, n).
struct GramPlan {
  int ntb;       // 64-wide column blocks
  int ntiles;    // upper-triangle output tiles
  int nchunk;    // sample chunks
  int64_t chunk; // samples per chunk (multiple of 16)
};
inline GramPlan gram_plan(int ncol, int64_t n) {
  GramPlan g;
  g.ntb = (ncol + 63) / 64;
  g.ntiles = g.ntb * (g.ntb + 1) / 2;
  int64_t nchunk = (2 * 148 + g.ntiles - 1) / g.ntiles;
  const int64_t cap = n / 512 > 1 ? n / 512 : 1;
  if (nchunk > cap) nchunk = cap;
  if (nchunk < 1) nchunk = 1;
  g.chunk = ((n + nchunk - 1) / nchunk + 15) / 16 * 16;
  g.nchunk = static_cast<int>((n + g.chunk - 1) / g.chunk);
  return g;
}
inline int64_t gram_scratch_doubles(int ncol, int64_t n) {
  const GramPlan g = gram_plan(ncol, n);
  return g.nchunk > 1 ? static_cast<int64_t>(g.nchunk) * g.ntiles * 64 * 64 : 0;
}
void launch_gram(const double* W, int64_t ldw, int64_t n, int ncol, double* C, int64_t ldc,
                 double* scratch, cudaStream_t s);

// k[p] = sum_{q != p} min(0, M_pq)^2 with M_pq = (H_q + E(p|q)) - (H_p + E(q|p)).
// errs[0..world): error keys gathered from every rank (world = 1: errs = err).
// KN (optional, d x d by variable): KN[act[p] * d + act[q]] = min(0, M_pq)^2 for every pair
// (the pruned rounds' knowledge, prune_kernels.cu).
void launch_kreduce(const double* epack, const double* H, int u, int nb, double* k,
                    unsigned long long* err, const unsigned long long* errs, int world,
                    const int* act, double* KN, int d, cudaStream_t s);

// ---- exact pruned search round (prune_kernels.cu) ----
// Row states: 0 pruned (k provably > k*), 1 alive, 2 top (full row from the start).
struct PruneArgs {
  const double* W;
  int64_t ldw;
  int64_t n;
  const double* C;
  int64_t ldc;
  const int* act;
  int u;
  int d;
  const double* H;              // [u] column entropies of the round
  double* Md;                   // [u * u] M_pq of evaluated pairs, NaN otherwise
  double* KN;                   // [d * d] last evaluated min(0, M)^2 by variable pair
  const int* state_in;          // [u]
  int* state_out;               // [u]
  double* L;                    // [u] partial k over the evaluated pairs
  unsigned long long* kstar;    // bits of min exact k over the top rows
  double* pk;                   // [u] predicted k (sum of KN over the active row)
  int* cand;                    // [u][4] strongest predicted partners of each row (ordered)
  int* rowsel;                  // [u * u] selected partner positions of each row, ascending
  int* off;                     // [u + 1] per-row counts -> exclusive offsets, off[u] = total
  int* crow;                    // [list / 32 + 1] row of each 32-entry chunk's first entry
  int* alive;                   // [1 + u] count, then the stage's surviving rows (any order)
  double* part;                 // [nseg][batch][4] segment partial sums
  int* work;                    // per-batch item counters (zeroed by the scan kernel)
  int* done;                    // [batch / 32] per-chunk finished-segment counters (self-resetting)
  int batch;                    // pairs per batch of the list kernel
  int seg_len;
  int nseg;
  int seg_major;                // pair-list item order: segment-major (1) or chunk-major (0)
  int fine_items;               // lists with fewer items split their segments (0: never)
  double top_ratio;             // > 0: one top row when its prediction < top_ratio x the runner-up's
  const double* g_exp;
  const double2* g_log;
  unsigned long long* err;
  int round;
  double* k;                    // [u] exact k of alive/top rows, +inf for pruned rows
  unsigned long long* evals;    // [1 + stages] list entries evaluated: total, per stage index
  int stage_idx;
  int k_begin;                  // list entries this launch evaluates: [k_begin, k_end)
  int k_end;                    // (k_end < 0: the whole list from k_begin)
  double* res;                  // multi-rank: M of the list entries, one slot per rank (all-gathered)
  int res_base;                 // this launch's first entry goes to res[res_base] (host-planned slices)
  int shard_world;              // > 0: slice of this rank planned on the device from the list length
  int shard_rank;
  int shard_slot;               // entries per rank slot in res
  int* stage_log;               // analysis (PLG_STAGE_LOG): [round][kMaxPruneStages] list lengths, or null
  PeerTable peers;              // n > 0: list entry k's M goes to res[k] of every rank (peer memory)
};
enum PruneStage : int { kStageProbe = 0, kStageRefine = 1, kStageFull = 2 };
void launch_prune_predict(const PruneArgs& a, cudaStream_t s);
void launch_prune_top(const PruneArgs& a, int R, cudaStream_t s);
// m: partners per row (probe: suspects per non-top row; refine: top-m predicted);
// beta > 0 (refine): deficit mode — predicted contributions reaching beta x the row's deficit
void launch_prune_select(const PruneArgs& a, int stage, int m, double beta, cudaStream_t s);
void launch_prune_scan(const PruneArgs& a, cudaStream_t s);
cudaError_t launch_prune_pairs(const PruneArgs& a, cudaStream_t s);  // cooperative launch result
// multi-rank: all ranks' results (res, `world` slots of `slot` entries; entry k of the list
// sits at (k / cnt) slot + k % cnt with cnt = ceil(total / world)) into Md / KN
// p2p_wait: peer-memory contexts, wait for every rank's signal of this stage first
void launch_prune_scatter(const PruneArgs& a, int world, int slot, cudaStream_t s, bool p2p_wait = false);
// pass 0: every row's partial k L[] and k* over the top rows; 1: alive rows' L[]; 2: exact k[]
// of the top and alive rows (+inf for pruned rows)
void launch_prune_bound(const PruneArgs& a, int pass, cudaStream_t s);
constexpr int kMaxPruneStages = 8;

// argmin over k (lowest position on ties), order/score bookkeeping, active-list compaction;
// round_k (optional): the winning k of each round; round_second (optional): the runner-up's
// k, with lb[p] standing in for rows whose k a pruned round left at +inf (near-tie guard).
void launch_commit(const double* k, const int* act_cur, int* act_nxt, int u, const int* col_var,
                   int* order, int round, double* scores, RoundState* rs,
                   const unsigned long long* err, cudaStream_t s, double* round_k = nullptr,
                   const double* lb = nullptr, double* round_second = nullptr);

// Rank-1 Schur update of the remaining Gram block: Cn_rs = C_rs - C_rm C_ms / C_mm (Cn == C:
// in place; else the next round's buffer of a ping-pong pair).
__host__ __device__ inline double gram_update_entry(double c_rs, double c_rm, double c_ms, double c_mm) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(c_rs, __ddiv_rn(__dmul_rn(c_rm, c_ms), c_mm));
#else
  return c_rs - (c_rm * c_ms) / c_mm;
#endif
}
void launch_update_gram(const double* C, double* Cn, int64_t ldc, const int* act_nxt, int ur, const RoundState* rs,
                        const unsigned long long* err, cudaStream_t s);


// Reference regress_out (ordering.cpp:178-211): raw columns, fresh means, bit-exact.
void launch_regress_out(const double* X, int64_t ldx, int64_t n, int exog, const int* remaining,
                        int r, double* out, int64_t ldo, int* zero_var_flag, cudaStream_t s);

// FP64 blocked Householder QR in echelon form (qr_kernels.cu): weights of DirectLiNGAM
// (every predecessor regression from one QR of the order-permuted centred design) and the
// VAR least squares. A (n x ncol, lda) is factored in place; thr[k]: a column whose residual
// norm is <= thr[k] is dependent (no reflector). qstate = {rank, dependent count}.
constexpr int kQrNB = 32;
void launch_qr_center(const double* X, int64_t ldx, int64_t n, const int* order, int ncol, int center, double* A,
                      int64_t lda, double* cn, cudaStream_t s);
void launch_qr_thr_prefix(const double* cn, int64_t n, int d, double* thr, int* qstate, cudaStream_t s);
void launch_qr_thr_design(const double* cn, int64_t n, int ncol, int ntot, double* thr, int* qstate, cudaStream_t s);
int64_t qr_scratch_doubles(int64_t n, int ncol);  // Yp + Z of the trailing updates
cudaError_t launch_qr_factor(double* A, int64_t lda, int64_t n, int ncol, const double* thr, int* qstate,
                             int* rbefore, int* rowcol, double* tau, int* dep, int* pinfo, double* T, double* Yp,
                             double* Z, cudaStream_t s);
cudaError_t launch_qr_solve(const double* A, int64_t lda, int ncol, int k_first, const int* rbefore, const int* rowcol,
                            double* coef, int64_t ldcoef, const int* order, double* B, int64_t ldb, cudaStream_t s);
cudaError_t launch_qr_mincorr(const double* coef, int64_t ldcoef, const int* rbefore, const int* rowcol,
                              const int* deps, const int* tg, const int* mcount, int ntg, const int* order, double* N,
                              int mmax, double* B, int64_t ldb, cudaStream_t s);

// VarLiNGAM front-end (var_kernels.cu): stacked design, normal equations, residuals.
void launch_build_var_design(const double* ts, int64_t ldt, int64_t n_rows, int d, int lag, double* A, int64_t lda,
                             int* nonfinite, cudaStream_t s);
void launch_var_resid(const double* A, int64_t lda, int64_t n_rows, int n_cols, int d, const double* B, double* E,
                      int64_t lde, cudaStream_t s);

// entropy_approx(u * scale) of one vector (kernels.cpp:123-148).
void launch_entropy_vec(const double* u, int64_t n, double scale, double* out, const double* g_exp,
                        const double2* g_log, cudaStream_t s);

// Test hook: evaluate lc/pdf element functions on a vector (custom and libdevice).
void launch_math_probe(const double* u, int64_t n, double* out, const double* g_exp,
                       const double2* g_log, cudaStream_t s);

}  // namespace plg

namespace plg {
__host__ __device__ inline int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
}  // namespace plg
