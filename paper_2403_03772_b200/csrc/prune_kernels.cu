// prune_kernels.cu — the exact pruned search round (branch and bound over candidates).
//
// causal_order only needs the round's argmin of k_p = sum_q min(0, M_pq)^2 (reference
// ordering.cpp:154-160), not every k. Every term is >= 0, so the sum over any subset of a
// row's pairs is a lower bound of k_p. A round therefore evaluates pairs in stages:
//
//   probe   full rows of the R candidates with the lowest predicted k (k* = the smallest of
//           their exact k) + each other row's T strongest predicted partners
//   refine  rows whose partial k has not passed k* evaluate their top-m predicted partners
//           (m = f u, one stage per fraction f)
//   full    rows still alive evaluate every remaining partner: exact k
//
// and a row is pruned as soon as its partial k exceeds k* (1 + 1e-9): the partial and the
// full sums are FP64 sums of the same non-negative terms, whose orders differ by at most
// u 2^-53 relative, so a pruned row's exact k is strictly larger than k* and it can neither
// win nor tie. The winner is the lowest-position argmin over the rows with exact k, which is
// the argmin of the full round. Every evaluated pair has the bits the exhaustive round gives
// it (same per-pair scales, element math and sample-segment reduction order), so the exact
// k of the surviving rows — the winner's included — are the exhaustive round's bits.
//
// Predictions come from KN (d x d, by variable): the last evaluated min(0, M_pq)^2 of every
// pair, filled completely by the exhaustive round 0 and refreshed with every evaluated pair
// afterwards. Removing one root changes most M_pq only slightly, so last round's strongest
// contributors prune a row after a few pairs (non-roots: usually one pair with an ancestor).
//
// Pair lists are built deterministically (per-row selection in ascending partner order +
// exclusive scan), and evaluated by a cooperative persistent kernel that streams batches of
// 32-pair chunks x sample segments and finalises each batch after a grid barrier, so the
// list length never has to reach the host.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "plg_async.cuh"
#include "plg_kernels.h"
#include "plg_math.cuh"
#include "plg_pair.cuh"

namespace cg = cooperative_groups;

namespace plg {

namespace {

constexpr unsigned long long kInfBits = 0x7ff0000000000000ull;
constexpr int kPredK = 4;  // predicted partners kept per row by prune_predict (probe suspects; R + T <= 4)
constexpr double kPruneSlack = 1e-9;  // relative margin over k* (>> u 2^-53)

__device__ __forceinline__ bool is_eval(double m) { return m == m; }  // NaN = not evaluated

__device__ __forceinline__ double kstar_threshold(const PruneArgs& a) {
  return __longlong_as_double(static_cast<long long>(*a.kstar)) * (1.0 + kPruneSlack);
}

// Partner order of the predictions: larger KN first, ties to the lower position.
__device__ __forceinline__ bool key_better(unsigned long long k1, int q1, unsigned long long k2, int q2) {
  return q2 < 0 || (q1 >= 0 && (k1 > k2 || (k1 == k2 && q1 < q2)));
}

// Lane-sorted top-K insertion (registers; K compile-time).
template <int K>
__device__ __forceinline__ void insert_key(unsigned long long (&bk)[K], int (&bq)[K], unsigned long long key, int q) {
  if (!key_better(key, q, bk[K - 1], bq[K - 1])) return;  // the common case: not in the lane's top K
#pragma unroll
  for (int i = 0; i < K; ++i) {
    if (key_better(key, q, bk[i], bq[i])) {
      const unsigned long long tk = bk[i];
      const int tq = bq[i];
      bk[i] = key, bq[i] = q;
      key = tk, q = tq;
    }
  }
}

// ---- predict: pk[p] = sum_q KN(p, q); the row's kPredK strongest predicted partners (the
// probe stage's suspects come from them); collinearity of every pair; state = alive ----
constexpr int kPredThreads = 128;  // 4 warps per row: enough loads in flight at ~2000 rows
__global__ void __launch_bounds__(kPredThreads) prune_predict_kernel(const PruneArgs a) {
  __shared__ double s_acc[kPredThreads / 32];
  __shared__ unsigned long long s_bk[kPredThreads / 32][kPredK];
  __shared__ int s_bq[kPredThreads / 32][kPredK];
  __shared__ int s_col[kPredThreads / 32];
  const int p = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int vp = a.act[p];
  const double* kn = a.KN + static_cast<int64_t>(vp) * a.d;
  const double* crow = a.C + static_cast<int64_t>(vp) * a.ldc;
  const double cii = crow[vp];
  double acc = 0.0;
  bool collinear = false;
  unsigned long long bk[kPredK];
  int bq[kPredK];
#pragma unroll
  for (int i = 0; i < kPredK; ++i) bk[i] = 0ull, bq[i] = -1;
  for (int q0 = threadIdx.x; q0 < a.u; q0 += 4 * kPredThreads) {
    int vq[4];
    double kv[4], cjj[4], cij[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // independent loads first
      const int q = q0 + kPredThreads * j;
      vq[j] = q < a.u ? a.act[q] : vp;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      kv[j] = kn[vq[j]];
      cjj[j] = a.C[static_cast<int64_t>(vq[j]) * a.ldc + vq[j]];
      cij[j] = crow[vq[j]];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int q = q0 + kPredThreads * j;
      if (q >= a.u) continue;
      acc += (q == p) ? 0.0 : kv[j];
      if (q != p) insert_key<kPredK>(bk, bq, static_cast<unsigned long long>(__double_as_longlong(kv[j])), q);
      // pair_scales' test (the exhaustive round checks every pair). Pairs with
      // C_ij^2 < C_ii C_jj (1 - 1e-6) have both residual variances > 0 whatever the rounding.
      if (q > p && !(cij[j] * cij[j] < cii * cjj[j] * (1.0 - 1e-6))) {
        double b1, v1, b2, v2;
        pair_vars(cii, cjj[j], cij[j], b1, v1, b2, v2);
        collinear |= pair_collinear(v1, v2);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  const bool wcol = __any_sync(0xffffffffu, collinear);
  // the warp's best kPredK (merge of the lanes' sorted lists)
#pragma unroll
  for (int r = 0; r < kPredK; ++r) {
    unsigned long long k = bk[0];
    int q = bq[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, k, o);
      const int oq = __shfl_xor_sync(0xffffffffu, q, o);
      if (key_better(ok, oq, k, q)) k = ok, q = oq;
    }
    if (lane == 0) s_bk[warp][r] = k, s_bq[warp][r] = q;
    if (q >= 0 && bq[0] == q) {
#pragma unroll
      for (int i = 0; i + 1 < kPredK; ++i) bk[i] = bk[i + 1], bq[i] = bq[i + 1];
      bk[kPredK - 1] = 0ull, bq[kPredK - 1] = -1;
    }
  }
  if (lane == 0) s_acc[warp] = acc, s_col[warp] = wcol;
  __syncthreads();
  if (warp != 0) return;
  // row totals in a fixed order; the row's best kPredK from the warps' lists
  unsigned long long k = 0ull;
  int q = -1;
  if (lane < (kPredThreads / 32) * kPredK) k = s_bk[lane / kPredK][lane % kPredK], q = s_bq[lane / kPredK][lane % kPredK];
  int* cand = a.cand + static_cast<int64_t>(p) * kPredK;
#pragma unroll
  for (int r = 0; r < kPredK; ++r) {
    unsigned long long bkk = k;
    int bqq = q;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, bkk, o);
      const int oq = __shfl_xor_sync(0xffffffffu, bqq, o);
      if (key_better(ok, oq, bkk, bqq)) bkk = ok, bqq = oq;
    }
    if (lane == 0) cand[r] = bqq;
    if (bqq >= 0 && q == bqq) k = 0ull, q = -1;
  }
  if (lane == 0) {
    double tot = 0.0;
    bool col = false;
    for (int w = 0; w < kPredThreads / 32; ++w) tot += s_acc[w], col |= (s_col[w] != 0);
    if (col) atomicMin(a.err, err_key(a.round, kErrPairCollinear, -1));
    a.pk[p] = tot;
    a.state_out[p] = 1;
    a.L[p] = 0.0;
  }
}

// ---- top: the R rows with the lowest pk (ties: lowest position) become full rows ----
// Each warp keeps its lanes' best R (insertion) and merges them by shuffles; warp 0 merges
// the warps' lists. Two block barriers in all.
constexpr int kTopThreads = 256;
constexpr int kMaxR = 16;

__device__ __forceinline__ bool pk_better(double v1, int p1, double v2, int p2) {
  return p2 < 0 || (p1 >= 0 && (v1 < v2 || (v1 == v2 && p1 < p2)));
}

// Merge the lanes' sorted lists (length kMaxR, first R used) into the warp's best R, in order.
__device__ __forceinline__ void warp_merge_best(double (&bv)[kMaxR], int (&bp)[kMaxR], int R, double* ov, int* op) {
  const int lane = threadIdx.x & 31;
  for (int r = 0; r < R; ++r) {
    double v = bv[0];
    int p = bp[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
      const int p2 = __shfl_xor_sync(0xffffffffu, p, o);
      if (pk_better(v2, p2, v, p)) v = v2, p = p2;
    }
    if (lane == 0) ov[r] = v, op[r] = p;
    if (p >= 0 && bp[0] == p) {
#pragma unroll
      for (int i = 0; i + 1 < kMaxR; ++i) bv[i] = bv[i + 1], bp[i] = bp[i + 1];
      bp[kMaxR - 1] = -1;
    }
  }
}

__device__ __forceinline__ void insert_best(double (&bv)[kMaxR], int (&bp)[kMaxR], int R, double v, int p) {
#pragma unroll
  for (int i = 0; i < kMaxR; ++i) {
    if (i < R && pk_better(v, p, bv[i], bp[i])) {
      const double tv = bv[i];
      const int tp = bp[i];
      bv[i] = v, bp[i] = p;
      v = tv, p = tp;
    }
  }
}

__global__ void __launch_bounds__(kTopThreads) prune_top_kernel(const PruneArgs a, int R) {
  __shared__ double sv[kTopThreads / 32][kMaxR];
  __shared__ int sp[kTopThreads / 32][kMaxR];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) *a.kstar = kInfBits;
  double bv[kMaxR];
  int bp[kMaxR];
#pragma unroll
  for (int i = 0; i < kMaxR; ++i) bv[i] = 0.0, bp[i] = -1;
  for (int p = threadIdx.x; p < a.u; p += kTopThreads) insert_best(bv, bp, R, a.pk[p], p);
  warp_merge_best(bv, bp, R, sv[warp], sp[warp]);
  __syncthreads();
  if (warp != 0) return;
#pragma unroll
  for (int i = 0; i < kMaxR; ++i) bv[i] = 0.0, bp[i] = -1;
  for (int w = lane; w < kTopThreads / 32; w += 32)
    for (int r = 0; r < R; ++r) insert_best(bv, bp, R, sv[w][r], sp[w][r]);
  __shared__ double fv[kMaxR];
  __shared__ int fp[kMaxR];
  warp_merge_best(bv, bp, R, fv, fp);
  __syncwarp();
  // a clear favourite (its predicted k below top_ratio x the runner-up's) gets the full row
  // alone; otherwise the R best do (k* must be tight for pruning to bite)
  int r_eff = R;
  if (a.top_ratio > 0.0 && R >= 2 && fp[1] >= 0 && fv[0] < a.top_ratio * fv[1]) r_eff = 1;
  if (lane < r_eff && fp[lane] >= 0) a.state_out[fp[lane]] = 2;
}

// ---- select: each row's partners for one stage, ascending, into rowsel[p * u + i] ----
constexpr int kSelThreads = 256;
constexpr int kBins = 2049;  // 0: known zero; 1 + biased exponent otherwise (1: unknown marker)
constexpr int kWSplit = 15;            // fixed-point weight = hi << 15 + lo
constexpr double kWMax = 134217727.0;  // 2^27 - 1: 8x the deficit target (2^24)

__device__ __forceinline__ int key_bin(double v) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return b == 0 ? 0 : 1 + static_cast<int>(b >> 52);
}

// Block-wide exclusive prefix of a predicate over one 256-wide chunk; returns the chunk total.
__device__ __forceinline__ int block_prefix(bool pred, int* s_warp, int& excl) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, pred);
  if (lane == 0) s_warp[warp] = __popc(bal);
  __syncthreads();
  int before = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kSelThreads / 32; ++w) {
    const int c = s_warp[w];
    before += (w < warp) ? c : 0;
    total += c;
  }
  excl = before + __popc(bal & ((1u << lane) - 1u));
  __syncthreads();
  return total;
}

// Refinement selection, two modes. Count mode (beta <= 0): the m partners with the largest
// predicted contribution. Deficit mode (beta > 0): partners in descending predicted
// contribution until their predicted sum reaches beta (thr - L_p), the amount the row's
// partial k still lacks to be pruned; if all its predictions together fall short, every
// remaining partner (the row is a contender and needs its exact k anyway). Selection works
// on exponent bins of the predicted value (2^k granularity) with fixed-point weights, so it
// is deterministic; inside the boundary bin partners are taken in ascending position.
// Refinement / full stages, step 1 (CTA of 128 threads per row): the row's partial k over
// its evaluated partners (a lower bound of k whatever the summation order; fixed block
// shape, so deterministic), the prune decision, and the compact list of surviving rows
// (its order is irrelevant: each row's selection depends on that row only).
constexpr int kRowThreads = 128;
__global__ void __launch_bounds__(kRowThreads) prune_rowl_kernel(const PruneArgs a) {
  __shared__ double s_red[kRowThreads / 32];
  const int p = blockIdx.x;
  const int u = a.u;
  const int st = a.state_in[p];
  if (st != 1) {
    if (threadIdx.x == 0) a.state_out[p] = st, a.off[p] = 0;
    return;
  }
  const double* md = a.Md + static_cast<int64_t>(p) * u;
  double acc = 0.0;
#pragma unroll 4
  for (int q = threadIdx.x; q < u; q += kRowThreads) {
    const double mi = md[q];
    if (q != p && is_eval(mi)) {
      const double c = (mi < 0.0) ? mi : 0.0;
      acc = __dadd_rn(acc, __dmul_rn(c, c));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double Lp = 0.0;
  for (int w = 0; w < kRowThreads / 32; ++w) Lp += s_red[w];
  const bool alive = Lp <= kstar_threshold(a);
  a.L[p] = Lp;
  a.state_out[p] = alive ? 1 : 0;
  a.off[p] = 0;  // the selection overwrites it for surviving rows
  if (alive) a.alive[1 + atomicAdd(a.alive, 1)] = p;
}

// Step 2 (CTA per surviving row, from the compact list; probe fallback: CTA per row).
__global__ void __launch_bounds__(kSelThreads) prune_select_kernel(const PruneArgs a, int stage, int m,
                                                                   double beta, int cache_keys) {
  __shared__ int hist[kBins];
  // per-bin fixed-point weight sums as two 32-bit halves (native shared atomics: a 64-bit
  // shared atomicAdd is a CAS loop, and hot bins made it the kernel's top stall)
  __shared__ unsigned int wlo[kBins], whi[kBins];
  auto wt = [&](int b) -> unsigned long long {
    return (static_cast<unsigned long long>(whi[b]) << kWSplit) + wlo[b];
  };
  __shared__ int s_warp[kSelThreads / 32];
  __shared__ int s_cut[2];  // boundary bin, entries of it to take
  __shared__ unsigned long long s_pw[kSelThreads];  // per-thread partial weights of its bins
  __shared__ int s_pn[kSelThreads];                 // ... and entry counts
  extern __shared__ double s_key[];  // cache_keys: per partner, its prediction or -1 (not eligible)
  const int u = a.u;
  const bool refine = (stage != kStageProbe);
  if (refine && static_cast<int>(blockIdx.x) >= *a.alive) return;
  const int p = refine ? a.alive[1 + blockIdx.x] : static_cast<int>(blockIdx.x);
  const int st = a.state_in[p];
  const double thr = refine ? kstar_threshold(a) : 0.0;
  const double Lp = refine ? a.L[p] : 0.0;
  const double* md = a.Md + static_cast<int64_t>(p) * u;
  const double* kn = a.KN + static_cast<int64_t>(a.act[p]) * a.d;
  const bool full = refine ? (stage == kStageFull) : (st == 2);
  if (!refine && threadIdx.x == 0) a.state_out[p] = st;
  // The row's predictions for its unevaluated partners, cached in shared memory (loads 8 per
  // thread at a time: the gather kn[act[q]] depends on act[q]).
  const bool cached = cache_keys && refine;
  if (cached) {
    constexpr int kB = 8;
    for (int q0 = threadIdx.x; q0 < u; q0 += kB * kSelThreads) {
      double mi[kB];
      int vq[kB];
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        const int q = q0 + j * kSelThreads;
        mi[j] = q < u ? md[q] : 0.0;
        vq[j] = q < u ? a.act[q] : 0;
      }
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        const int q = q0 + j * kSelThreads;
        if (q < u) s_key[q] = (q == p || is_eval(mi[j])) ? -1.0 : kn[vq[j]];
      }
    }
    __syncthreads();
  }
  // A pair of two full rows is listed twice in the full stage (both rows are still alive,
  // rare); its two evaluations have identical bits and the same writes.
  auto eligible = [&](int q) -> bool {
    if (cached) return s_key[q] >= 0.0;
    if (q == p || is_eval(md[q])) return false;
    if (stage == kStageProbe) return full ? !(a.state_in[q] == 2 && q < p) : a.state_in[q] != 2;
    return true;
  };
  auto key_of = [&](int q) -> double { return cached ? s_key[q] : kn[a.act[q]]; };
  // Modes: count (beta <= 0): the m strongest; deficit (m <= 0): strongest until their
  // predicted sum reaches beta x deficit, else all; hybrid (both): the deficit cut when it
  // needs fewer than m partners, else the m strongest.
  const bool deficit = beta > 0.0;
  constexpr double kOne = 16777216.0;  // fixed-point unit of the deficit target (2^24)
  const double target = fmax(beta * (thr - Lp), thr * 1e-6);
  const double wscale = deficit ? kOne / target : 0.0;
  int cut_bin = -1, cut_take = 0;  // full: every eligible partner
  if (!full) {
    for (int i = threadIdx.x; i < kBins; i += kSelThreads) hist[i] = 0, wlo[i] = 0u, whi[i] = 0u;
    __syncthreads();
    for (int q0 = 0; q0 < u; q0 += kSelThreads) {  // warp-aggregated bin increments
      const int q = q0 + threadIdx.x;
      const bool e = q < u && eligible(q);
      const double v = e ? key_of(q) : 0.0;
      const int b = e ? key_bin(v) : -1;
      const unsigned grp = __match_any_sync(0xffffffffu, b);
      const int leader = __ffs(grp) - 1;
      if (e && (threadIdx.x & 31) == leader) atomicAdd(&hist[b], __popc(grp));
      if (deficit && e) {
        // weights clamped at kWMax (8x the target): one element that alone reaches the target
        // gives the same cut bin; the two halves' sums stay below 2^32 for u < 2^17
        const unsigned long long w = static_cast<unsigned long long>(fmin(v * wscale, kWMax));
        atomicAdd(&wlo[b], static_cast<unsigned int>(w & ((1ull << kWSplit) - 1)));
        atomicAdd(&whi[b], static_cast<unsigned int>(w >> kWSplit));
      }
    }
    __syncthreads();
    // Partial sums of kPerT consecutive bins per thread (top-down), in parallel: warp 0's cut
    // search then walks 8 thread partials and at most kPerT bins instead of 65 bins per lane
    // (it held the other warps at the barrier for ~20% of the kernel). Integer sums: the cut
    // does not depend on the partition.
    constexpr int kPerT = (kBins + kSelThreads - 1) / kSelThreads;  // 9
    {
      const int hiT = kBins - 1 - static_cast<int>(threadIdx.x) * kPerT;
      unsigned long long pw = 0;
      int pn = 0;
      for (int b = hiT; b > hiT - kPerT && b >= 0; --b) {
        if (deficit) pw += wt(b);
        pn += hist[b];
      }
      s_pw[threadIdx.x] = pw;
      s_pn[threadIdx.x] = pn;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // Suffix scan from the top bin (warp 0): the bin where the cumulative weight reaches
      // need; returns false when the total falls short. cnt_above = entries in higher bins.
      auto find_cut = [&](bool weighted, unsigned long long need_total, int& bin, int& take, int& cnt_above) -> bool {
        const int lane = threadIdx.x;
        constexpr int kT = kSelThreads / 32;  // thread partials per lane
        unsigned long long own = 0;
        int own_n = 0;
#pragma unroll
        for (int j = 0; j < kT; ++j) {
          own += weighted ? s_pw[lane * kT + j] : static_cast<unsigned long long>(s_pn[lane * kT + j]);
          own_n += s_pn[lane * kT + j];
        }
        unsigned long long incl = own;
        int incl_n = own_n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
          const int vn = __shfl_up_sync(0xffffffffu, incl_n, o);
          if (lane >= o) incl += v, incl_n += vn;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, incl >= need_total);
        if (hit == 0) return false;
        const int src = __ffs(hit) - 1;
        int r_bin = 0, r_take = 0, r_cnt = 0;
        if (lane == src) {
          unsigned long long cum = incl - own;
          int cn = incl_n - own_n;
          int t = lane * kT;
          for (;; ++t) {  // the thread partial that reaches need
            const unsigned long long wt_t = weighted ? s_pw[t] : static_cast<unsigned long long>(s_pn[t]);
            if (cum + wt_t >= need_total) break;
            cum += wt_t;
            cn += s_pn[t];
          }
          int b = kBins - 1 - t * kPerT;
          for (;;) {  // the bin within it
            const unsigned long long wb = weighted ? wt(b) : static_cast<unsigned long long>(hist[b]);
            if (cum + wb >= need_total) break;
            cum += wb;
            cn += hist[b];
            --b;
          }
          const unsigned long long need = need_total - cum;  // > 0, <= the bin's weight
          r_bin = b;
          r_take = weighted ? static_cast<int>((need * static_cast<unsigned long long>(hist[b]) + wt(b) - 1) / wt(b))
                            : static_cast<int>(need);
          r_cnt = cn;
        }
        bin = __shfl_sync(0xffffffffu, r_bin, src);
        take = __shfl_sync(0xffffffffu, r_take, src);
        cnt_above = __shfl_sync(0xffffffffu, r_cnt, src);
        return true;
      };
      int bin = -1, take = 0, above = 0;
      bool done = false;
      if (deficit && find_cut(true, static_cast<unsigned long long>(kOne), bin, take, above))
        done = (m <= 0) || (above + take < m);  // hybrid: keep the deficit cut only if smaller
      else if (deficit && m <= 0)
        bin = -1, take = 0, done = true;  // pure deficit mode, prediction short: every partner
      if (!done && !find_cut(false, static_cast<unsigned long long>(m), bin, take, above)) bin = -1, take = 0;
      if (threadIdx.x == 0) s_cut[0] = bin, s_cut[1] = take;
    }
    __syncthreads();
    cut_bin = s_cut[0];
    cut_take = s_cut[1];
  }
  // Emit in ascending q: bins above the cut, then the first cut_take of the cut bin. Each warp
  // owns a contiguous range of partners: it counts its selections, one block barrier gives
  // the warps' offsets, then it writes its range in order with ballots (no further barrier).
  int* out = a.rowsel + static_cast<int64_t>(p) * u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarps = kSelThreads / 32;
  const int span = ((u + kWarps - 1) / kWarps + 31) & ~31;
  const int q_lo = warp * span, q_hi = min(u, q_lo + span);
  auto classify = [&](int q, bool& above, bool& in_cut) {
    above = in_cut = false;
    if (q < q_hi && eligible(q)) {
      if (cut_bin < 0) {
        above = true;
      } else {
        const int b = key_bin(key_of(q));
        above = b > cut_bin;
        in_cut = (b == cut_bin);
      }
    }
  };
  int n_above = 0, n_cut = 0;
  for (int base = q_lo; base < q_hi; base += 32) {
    bool ab, ic;
    classify(base + lane, ab, ic);
    n_above += __popc(__ballot_sync(0xffffffffu, ab));
    n_cut += __popc(__ballot_sync(0xffffffffu, ic));
  }
  __shared__ int s_above[kWarps], s_cut_n[kWarps];
  if (lane == 0) s_above[warp] = n_above, s_cut_n[warp] = n_cut;
  __syncthreads();
  int cut_seen = 0, out_before = 0, written = 0, cut_before = 0;
  for (int w = 0; w < kWarps; ++w) {  // warp w takes the cut-bin entries ranked [cut_seen, ...)
    const int take_w = max(0, min(s_cut_n[w], cut_take - cut_seen));
    if (w < warp) out_before += s_above[w] + take_w, cut_before += s_cut_n[w];
    written += s_above[w] + take_w;
    cut_seen += s_cut_n[w];
  }
  int pos = out_before, cut_rank = cut_before;
  for (int base = q_lo; base < q_hi; base += 32) {
    bool ab, ic;
    classify(base + lane, ab, ic);
    const unsigned lt = (1u << lane) - 1u;
    const unsigned bc = __ballot_sync(0xffffffffu, ic);
    const bool sel = ab || (ic && cut_rank + __popc(bc & lt) < cut_take);
    const unsigned bs = __ballot_sync(0xffffffffu, sel);
    if (sel) out[pos + __popc(bs & lt)] = base + lane;
    pos += __popc(bs);
    cut_rank += __popc(bc);
  }
  if (threadIdx.x == 0) a.off[p] = written;
}

// ---- probe select (warp per row): top rows take every partner (a pair of two top rows
// belongs to the lower row), other rows their T strongest predicted partners among the
// non-top rows (largest KN, ties to the lowest position) ----
constexpr int kMaxT = 8;


__global__ void __launch_bounds__(256) prune_probe_select_kernel(const PruneArgs a, int T) {
  const int p = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= a.u) return;
  const int u = a.u;
  const int st = a.state_in[p];
  int* out = a.rowsel + static_cast<int64_t>(p) * u;
  if (lane == 0) a.state_out[p] = st;
  if (st == 2) {
    int written = 0;
    for (int base = 0; base < u; base += 32) {
      const int q = base + lane;
      const bool sel = q < u && q != p && !(q < p && a.state_in[q] == 2);
      const unsigned bal = __ballot_sync(0xffffffffu, sel);
      if (sel) out[written + __popc(bal & ((1u << lane) - 1u))] = q;
      written += __popc(bal);
    }
    if (lane == 0) a.off[p] = written;
    return;
  }
  {  // the T strongest non-top partners from predict's candidate list (kPredK >= T + R)
    const int* cand = a.cand + static_cast<int64_t>(p) * kPredK;
    int sel[kMaxT];
    int nsel = 0, seen = 0;
    for (int i = 0; i < kPredK && nsel < T; ++i) {
      const int q = cand[i];
      if (q < 0) break;
      ++seen;
      if (a.state_in[q] != 2) sel[nsel++] = q;
    }
    if (nsel == T || seen < kPredK) {  // complete (or the row has fewer partners): done
      if (lane == 0) {
        for (int i = 1; i < nsel; ++i)
          for (int j = i; j > 0 && sel[j] < sel[j - 1]; --j) {
            const int t = sel[j];
            sel[j] = sel[j - 1];
            sel[j - 1] = t;
          }
        for (int i = 0; i < nsel; ++i) out[i] = sel[i];
        a.off[p] = nsel;
      }
      return;
    }
  }
  const double* kn = a.KN + static_cast<int64_t>(a.act[p]) * a.d;
  unsigned long long bk[kMaxT];
  int bq[kMaxT];
#pragma unroll
  for (int i = 0; i < kMaxT; ++i) bk[i] = 0ull, bq[i] = -1;
  for (int q0 = lane; q0 < u; q0 += 128) {
    unsigned long long keys[4];
    bool ok[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // independent loads first
      const int q = q0 + 32 * j;
      ok[j] = q < u && q != p && a.state_in[q] != 2;
      keys[j] = ok[j] ? static_cast<unsigned long long>(__double_as_longlong(kn[a.act[q]])) : 0ull;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
    if (!ok[j]) continue;
    unsigned long long key = keys[j];
    int qq = q0 + 32 * j;
#pragma unroll
    for (int i = 0; i < kMaxT; ++i) {  // insertion into the lane's sorted list
      if (i < T && key_better(key, qq, bk[i], bq[i])) {
        const unsigned long long tk = bk[i];
        const int tq = bq[i];
        bk[i] = key, bq[i] = qq;
        key = tk, qq = tq;
      }
    }
    }
  }
  int sel[kMaxT];
  int nsel = 0;
#pragma unroll
  for (int r = 0; r < kMaxT; ++r) {
    if (r >= T) break;
    unsigned long long k = bk[0];
    int q = bq[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, k, o);
      const int oq = __shfl_xor_sync(0xffffffffu, q, o);
      if (key_better(ok, oq, k, q)) k = ok, q = oq;
    }
    if (q < 0) break;  // fewer than T partners
    sel[r] = q;
    nsel = r + 1;
    if (bq[0] == q) {  // the owner pops its head
#pragma unroll
      for (int i = 0; i + 1 < kMaxT; ++i) bk[i] = bk[i + 1], bq[i] = bq[i + 1];
      bk[kMaxT - 1] = 0ull, bq[kMaxT - 1] = -1;
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 1; i < kMaxT; ++i)  // ascending partner order
      for (int j = i; j > 0 && j < nsel && sel[j] < sel[j - 1]; --j) {
        const int t = sel[j];
        sel[j] = sel[j - 1];
        sel[j - 1] = t;
      }
    for (int i = 0; i < nsel; ++i) out[i] = sel[i];
    a.off[p] = nsel;
  }
}

// ---- scan: off[0..u) counts -> exclusive offsets, off[u] = total ----
__global__ void __launch_bounds__(1024) prune_scan_kernel(const PruneArgs a) {
  __shared__ int s_w[32];
  __shared__ int s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < a.u; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = (i < a.u) ? a.off[i] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += t;
      }
      s_w[lane] = w;
    }
    __syncthreads();
    const int excl = s_carry + (warp ? s_w[warp - 1] : 0) + incl - v;
    if (i < a.u) a.off[i] = excl;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += s_w[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.off[a.u] = s_carry;
    atomicAdd(a.evals, static_cast<unsigned long long>(s_carry));
    atomicAdd(a.evals + 1 + a.stage_idx, static_cast<unsigned long long>(s_carry));
    if (a.stage_log) a.stage_log[a.round * kMaxPruneStages + a.stage_idx] = s_carry;
  }
  for (int b = threadIdx.x; b <= s_carry / a.batch; b += blockDim.x) a.work[b] = 0;  // fetch counters
  if (threadIdx.x == 0) *a.alive = 0;  // the next stage's surviving-row list starts empty
  __syncthreads();  // every offset visible to the block
  const int total = s_carry;
  for (int p = threadIdx.x; p < a.u; p += blockDim.x) {  // chunk -> row of its first entry
    const int b = a.off[p], e = (p + 1 < a.u) ? a.off[p + 1] : total;
    for (int c = (b + 31) >> 5; c < ((e + 31) >> 5); ++c) a.crow[c] = p;
  }
}

// ---- pairs: cooperative persistent evaluation of the list ----
constexpr int kListThreads = 256;
constexpr int kMinSegLen = 32;  // finest sample segment of a short list (a multiple of 4)
constexpr int64_t kFineMaxN = 4096;  // short columns: few segments per pair, so short lists have few items

// Entry k of the stage's list: the row holding the entry's 32-chunk start (chunk_row, from the
// scan), then forward over rows that end before k (rows with zero entries share offsets).
__device__ __forceinline__ void list_entry(const PruneArgs& a, int k, int& p, int& q) {
  p = a.crow[k >> 5];
  while (p + 1 < a.u && a.off[p + 1] <= k) ++p;
  q = a.rowsel[static_cast<int64_t>(p) * a.u + (k - a.off[p])];
}

template <bool kClampA, typename Tab>
__device__ __forceinline__ void ede2(double xa, double ya, double s1, double bs1, double s2, double bs2,
                                     EdeAcc& acc1, EdeAcc& acc2, const Tab& tp) {
  ede_accumulate<kClampA>(fma(ya, -bs1, xa * s1), acc1, tp);
  ede_accumulate<kClampA>(fma(xa, -bs2, ya * s2), acc2, tp);
}

// One pair's two residual directions over samples [t0, t1) (t0 a multiple of 4), samples in
// ascending order per direction. Loads go straight to registers with a software prefetch:
// kVar 0: 4 samples per step, 1 step ahead; 1: 2 samples per step, 2 steps ahead;
// 2: 4 samples per step, 2 steps ahead.
template <bool kClampA, int kVar, typename Tab>
__device__ __forceinline__ void eval_segment(const double* wi, const double* wj, int64_t t0, int64_t t1, double s1,
                                             double bs1, double s2, double bs2, EdeAcc& acc1, EdeAcc& acc2,
                                             const Tab& tp) {
  auto ld = [](const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); };
  int64_t t = t0;
  if (kVar == 5) {  // variant 0 with 256-bit loads
    const int nstep = static_cast<int>((t1 - t) >> 2);
    if (nstep > 0) {
      const double* pi = wi + t;
      const double* pj = wj + t;
      double4 x = ldg256(pi), y = ldg256(pj);
#pragma unroll 1
      for (int i = 1; i <= nstep; ++i) {
        const double4 cx = x, cy = y;
        pi += 4;
        pj += 4;
        if (i < nstep) x = ldg256(pi), y = ldg256(pj);
        ede2<kClampA>(cx.x, cy.x, s1, bs1, s2, bs2, acc1, acc2, tp);
        ede2<kClampA>(cx.y, cy.y, s1, bs1, s2, bs2, acc1, acc2, tp);
        ede2<kClampA>(cx.z, cy.z, s1, bs1, s2, bs2, acc1, acc2, tp);
        ede2<kClampA>(cx.w, cy.w, s1, bs1, s2, bs2, acc1, acc2, tp);
      }
      t += 4 * static_cast<int64_t>(nstep);
    }
  } else if (kVar == 0) {
    // pointer increments and a 32-bit step count keep the address arithmetic out of the
    // register-starved loop (index arithmetic was rematerialised every step)
    const int nstep = static_cast<int>((t1 - t) >> 2);
    if (nstep > 0) {
      const double2* pi = reinterpret_cast<const double2*>(wi + t);
      const double2* pj = reinterpret_cast<const double2*>(wj + t);
      double2 xa = __ldg(pi), xb = __ldg(pi + 1), ya = __ldg(pj), yb = __ldg(pj + 1);
#pragma unroll 1
      for (int i = 1; i <= nstep; ++i) {
        const double2 cxa = xa, cxb = xb, cya = ya, cyb = yb;
        pi += 2;
        pj += 2;
        if (i < nstep) xa = __ldg(pi), xb = __ldg(pi + 1), ya = __ldg(pj), yb = __ldg(pj + 1);
        ede2<kClampA>(cxa.x, cya.x, s1, bs1, s2, bs2, acc1, acc2, tp);
        ede2<kClampA>(cxa.y, cya.y, s1, bs1, s2, bs2, acc1, acc2, tp);
        ede2<kClampA>(cxb.x, cyb.x, s1, bs1, s2, bs2, acc1, acc2, tp);
        ede2<kClampA>(cxb.y, cyb.y, s1, bs1, s2, bs2, acc1, acc2, tp);
      }
      t += 4 * static_cast<int64_t>(nstep);
    }
  } else if (kVar == 1) {  // 2 samples per step, loads 2 steps ahead
    const int nstep = static_cast<int>((t1 - t) >> 1);
    if (nstep > 0) {
      const double2* pi = reinterpret_cast<const double2*>(wi + t);
      const double2* pj = reinterpret_cast<const double2*>(wj + t);
      double2 x0 = __ldg(pi), y0 = __ldg(pj), x1 = x0, y1 = y0;
      if (nstep > 1) x1 = __ldg(pi + 1), y1 = __ldg(pj + 1);
#pragma unroll 1
      for (int i = 2; i < nstep + 2; ++i) {
        const double2 cx = x0, cy = y0;
        x0 = x1, y0 = y1;
        if (i < nstep) x1 = __ldg(pi + i), y1 = __ldg(pj + i);
        ede2<kClampA>(cx.x, cy.x, s1, bs1, s2, bs2, acc1, acc2, tp);
        ede2<kClampA>(cx.y, cy.y, s1, bs1, s2, bs2, acc1, acc2, tp);
      }
      t += 2 * static_cast<int64_t>(nstep);
    }
  } else {  // 4 samples per step, loads 2 steps ahead
    const int nstep = static_cast<int>((t1 - t) >> 2);
    if (nstep > 0) {
      const double2* pi = reinterpret_cast<const double2*>(wi + t);
      const double2* pj = reinterpret_cast<const double2*>(wj + t);
      double2 xa = __ldg(pi), xb = __ldg(pi + 1), ya = __ldg(pj), yb = __ldg(pj + 1);
      double2 xc = xa, xd = xb, yc = ya, yd = yb;
      if (nstep > 1) xc = __ldg(pi + 2), xd = __ldg(pi + 3), yc = __ldg(pj + 2), yd = __ldg(pj + 3);
#pragma unroll 1
      for (int i = 2; i < nstep + 2; ++i) {
        const double2 cxa = xa, cxb = xb, cya = ya, cyb = yb;
        xa = xc, xb = xd, ya = yc, yb = yd;
        if (i < nstep) xc = __ldg(pi + 2 * i), xd = __ldg(pi + 2 * i + 1), yc = __ldg(pj + 2 * i), yd = __ldg(pj + 2 * i + 1);
        ede2<kClampA>(cxa.x, cya.x, s1, bs1, s2, bs2, acc1, acc2, tp);
        ede2<kClampA>(cxa.y, cya.y, s1, bs1, s2, bs2, acc1, acc2, tp);
        ede2<kClampA>(cxb.x, cyb.x, s1, bs1, s2, bs2, acc1, acc2, tp);
        ede2<kClampA>(cxb.y, cyb.y, s1, bs1, s2, bs2, acc1, acc2, tp);
      }
      t += 4 * static_cast<int64_t>(nstep);
    }
  }
  for (; t < t1; ++t) ede2<kClampA>(wi[t], wj[t], s1, bs1, s2, bs2, acc1, acc2, tp);
}

// Variant 0's loop with the first step already loaded by the caller (kVar 4: the item's
// first data loads are issued before the pair's scales are computed, so their latency
// overlaps the Gram loads, divisions and square roots instead of following them).
template <bool kClampA, typename Tab>
__device__ __forceinline__ void eval_segment_pre(const double* wi, const double* wj, int64_t t0, int64_t t1, double s1,
                                                 double bs1, double s2, double bs2, EdeAcc& acc1, EdeAcc& acc2,
                                                 const Tab& tp, double2 xa, double2 xb, double2 ya, double2 yb) {
  int64_t t = t0;
  const int nstep = static_cast<int>((t1 - t) >> 2);
  if (nstep > 0) {
    const double2* pi = reinterpret_cast<const double2*>(wi + t);
    const double2* pj = reinterpret_cast<const double2*>(wj + t);
#pragma unroll 1
    for (int i = 1; i <= nstep; ++i) {
      const double2 cxa = xa, cxb = xb, cya = ya, cyb = yb;
      pi += 2;
      pj += 2;
      if (i < nstep) xa = __ldg(pi), xb = __ldg(pi + 1), ya = __ldg(pj), yb = __ldg(pj + 1);
      ede2<kClampA>(cxa.x, cya.x, s1, bs1, s2, bs2, acc1, acc2, tp);
      ede2<kClampA>(cxa.y, cya.y, s1, bs1, s2, bs2, acc1, acc2, tp);
      ede2<kClampA>(cxb.x, cyb.x, s1, bs1, s2, bs2, acc1, acc2, tp);
      ede2<kClampA>(cxb.y, cyb.y, s1, bs1, s2, bs2, acc1, acc2, tp);
    }
    t += 4 * static_cast<int64_t>(nstep);
  }
  for (; t < t1; ++t) ede2<kClampA>(wi[t], wj[t], s1, bs1, s2, bs2, acc1, acc2, tp);
}

// M_pq and M_qp = -M_pq into the round's table; KN (the next rounds' predictions) gets
// min(0, M)^2 in both directions.
__device__ __forceinline__ void store_pair(const PruneArgs& a, int p, int q, double mpq) {
  a.Md[static_cast<int64_t>(p) * a.u + q] = mpq;
  a.Md[static_cast<int64_t>(q) * a.u + p] = -mpq;
  const int vp = a.act[p], vq = a.act[q];
  const double cp = mpq < 0.0 ? mpq : 0.0, cq = mpq > 0.0 ? -mpq : 0.0;
  a.KN[static_cast<int64_t>(vp) * a.d + vq] = __dmul_rn(cp, cp);
  a.KN[static_cast<int64_t>(vq) * a.d + vp] = __dmul_rn(cq, cq);
}

// Finalise one 32-pair chunk once all its sample segments are in: segments in ascending
// order (finalize_kernel's order), both entropies, then M_pq and M_qp = -M_pq.
__device__ __forceinline__ void finalize_chunk(const PruneArgs& a, const double* part, int base, int m, int chunk,
                                               int lane, int kb) {
  const int kk = chunk * 32 + lane;
  if (kk >= m) return;
  int p, q;
  list_entry(a, base + kk, p, q);
  double l1 = 0.0, p1 = 0.0, l2 = 0.0, p2 = 0.0;
  const double2* src = reinterpret_cast<const double2*>(part + static_cast<int64_t>(kk) * 4);
  const int64_t stride = static_cast<int64_t>(a.batch) * 2;  // double2 per segment
#pragma unroll 8
  for (int s = 0; s < a.nseg; ++s) {  // loads run ahead; the adds stay in ascending order
    const double2 v1 = __ldcg(src);  // written by other SMs: bypass L1
    const double2 v2 = __ldcg(src + 1);
    l1 += v1.x;
    p1 += v1.y;
    l2 += v2.x;
    p2 += v2.y;
    src += stride;
  }
  const double inv_n = 1.0 / static_cast<double>(a.n);
  const double e_pq = entropy_from_sums(l1, p1, inv_n);  // E(p | q)
  const double e_qp = entropy_from_sums(l2, p2, inv_n);  // E(q | p)
  // ordering.cpp:93-94 (kreduce_kernel's expression); M_qp = -M_pq exactly
  const double mpq = (a.H[q] + e_pq) - (a.H[p] + e_qp);
  store_pair(a, p, q, mpq);
  if (a.res) {
    if (a.peers.n > 0) {  // peer memory: entry k of the stage list at res[k] of every rank
      peer_store(a.peers, &a.res[base + kk], mpq);  // published by p2p_signal after this kernel
    } else {
      a.res[a.res_base + (base + kk - kb)] = mpq;  // multi-rank (NCCL): this rank's slot
    }
  }
}

__device__ __forceinline__ void finalize_chunk_fine(const PruneArgs& a, const double* part, int base, int m, int chunk,
                                               int lane, int kb, int nseg, int64_t pstride) {
  const int kk = chunk * 32 + lane;
  if (kk >= m) return;
  int p, q;
  list_entry(a, base + kk, p, q);
  double l1 = 0.0, p1 = 0.0, l2 = 0.0, p2 = 0.0;
  const double2* src = reinterpret_cast<const double2*>(part + static_cast<int64_t>(kk) * 4);
  const int64_t stride = pstride * 2;  // double2 per segment
#pragma unroll 8
  for (int s = 0; s < nseg; ++s) {  // loads run ahead; the adds stay in ascending order
    const double2 v1 = __ldcg(src);  // written by other SMs: bypass L1
    const double2 v2 = __ldcg(src + 1);
    l1 += v1.x;
    p1 += v1.y;
    l2 += v2.x;
    p2 += v2.y;
    src += stride;
  }
  const double inv_n = 1.0 / static_cast<double>(a.n);
  const double e_pq = entropy_from_sums(l1, p1, inv_n);  // E(p | q)
  const double e_qp = entropy_from_sums(l2, p2, inv_n);  // E(q | p)
  // ordering.cpp:93-94 (kreduce_kernel's expression); M_qp = -M_pq exactly
  const double mpq = (a.H[q] + e_pq) - (a.H[p] + e_qp);
  store_pair(a, p, q, mpq);
  if (a.res) {
    if (a.peers.n > 0) {  // peer memory: entry k of the stage list at res[k] of every rank
      peer_store(a.peers, &a.res[base + kk], mpq);  // published by p2p_signal after this kernel
    } else {
      a.res[a.res_base + (base + kk - kb)] = mpq;  // multi-rank (NCCL): this rank's slot
    }
  }
}

// Work items (chunk of 32 list entries, sample segment) are fetched dynamically, chunk-major;
// the warp completing a chunk's last segment finalises it, so a batch needs no grid barrier.
// Lists longer than one batch (part-buffer capacity) run batch after batch with a grid
// barrier between them (the kernel is launched cooperatively).
template <bool kClampA, int kVar>
__global__ void __launch_bounds__(kListThreads, 2) prune_pairs_kernel(const PruneArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const TabAddr tp = load_tables_aligned(smem, a.g_exp, a.g_log, lane);
  __syncthreads();
  cg::grid_group grid = cg::this_grid();
  const bool skip = (*a.err != kNoError);  // only skips work: every CTA still meets the barriers
  // this launch's share of the list: [kb, ke) — host-planned (k_end < 0: to the end of the
  // list), or this rank's slice of ceil(total / shard_world) entries planned here
  int kb = a.k_begin, ke = a.k_end >= 0 ? a.k_end : a.off[a.u];
  if (a.shard_world > 0) {
    const int tot = a.off[a.u];
    const int cnt = (tot + a.shard_world - 1) / a.shard_world;
    kb = min(tot, a.shard_rank * cnt);
    ke = min(tot, (a.shard_rank + 1) * cnt);
    if (cnt > a.shard_slot) {  // the host-side slot bound broke: ranks would overwrite each other's slots
      if (blockIdx.x == 0 && threadIdx.x == 0) atomicMin(a.err, err_key(0, kErrInternal, -1));
      ke = kb;
    }
  }
  const int total = ke - kb;
  const int nbatch = (total + a.batch - 1) / a.batch;
  for (int b = 0; b < nbatch; ++b) {
    if (b > 0) grid.sync();  // every chunk of batch b - 1 is finalised: the part slab is free
    const int base = kb + b * a.batch;
    const int m = min(a.batch, total - b * a.batch);
    const int chunks = (m + 31) / 32;
    const int items = chunks * a.nseg;
    int it = 0;
    if (lane == 0 && !skip) it = atomicAdd(&a.work[b], 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    while (!skip && it < items) {
      int chunk, seg;
      if (a.seg_major) {  // a sample window of every chunk at a time: column slices stay in L2
        seg = it / chunks;
        chunk = it - seg * chunks;
      } else {  // a chunk's segments back to back: its partial sums stay in L2
        chunk = it / a.nseg;
        seg = it - chunk * a.nseg;
      }
      const int kk = chunk * 32 + lane;
      if (kk < m) {
        int p, q;
        list_entry(a, base + kk, p, q);
        const int ci = a.act[p], cj = a.act[q];
        const double* wi = a.W + static_cast<int64_t>(ci) * a.ldw;
        const double* wj = a.W + static_cast<int64_t>(cj) * a.ldw;
        const int64_t t0 = static_cast<int64_t>(seg) * a.seg_len;  // multiple of 4: 32-byte aligned
        const int64_t t1 = lmin(a.n, t0 + a.seg_len);
        EdeAcc acc1, acc2;
        if (kVar == 4) {
          double2 xa = make_double2(0.0, 0.0), xb = xa, ya = xa, yb = xa;
          if (t0 + 3 < t1) {
            const double2* pi = reinterpret_cast<const double2*>(wi + t0);
            const double2* pj = reinterpret_cast<const double2*>(wj + t0);
            xa = __ldg(pi), xb = __ldg(pi + 1), ya = __ldg(pj), yb = __ldg(pj + 1);
          }
          double s1, bs1, s2, bs2;
          pair_scales(a.C, a.ldc, ci, cj, s1, bs1, s2, bs2);  // collinear pairs: zeros (flagged by predict)
          eval_segment_pre<kClampA>(wi, wj, t0, t1, s1, bs1, s2, bs2, acc1, acc2, tp, xa, xb, ya, yb);
        } else {
          double s1, bs1, s2, bs2;
          pair_scales(a.C, a.ldc, ci, cj, s1, bs1, s2, bs2);  // collinear pairs: zeros (flagged by predict)
          eval_segment<kClampA, kVar>(wi, wj, t0, t1, s1, bs1, s2, bs2, acc1, acc2, tp);
        }
        double2* dst = reinterpret_cast<double2*>(a.part + (static_cast<int64_t>(seg) * a.batch + kk) * 4);
        __stcg(dst, make_double2(acc_lc(acc1), acc_pdf(acc1)));
        __stcg(dst + 1, make_double2(acc_lc(acc2), acc_pdf(acc2)));
      }
      fence_release_gpu();  // release this segment's partials before counting it (no L1 invalidation)
      __syncwarp();
      // the segment count and the next item's fetch go out together: one L2 round trip per item
      int last = 0, next = 0;
      if (lane == 0) {
        last = (atomicAdd(&a.done[chunk], 1) == a.nseg - 1);
        next = atomicAdd(&a.work[b], 1);
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      it = __shfl_sync(0xffffffffu, next, 0);
      if (last) {
        fence_acquire_gpu();  // acquire the other segments' partials
        finalize_chunk(a, a.part, base, m, chunk, lane, kb);
        if (lane == 0) a.done[chunk] = 0;  // ready for the next batch / launch
      }
    }
  }
}

// The same kernel for short columns (n <= kFineMaxN, where short lists have few items): the
// list's segmentation may be refined at run time (below). A separate kernel because the
// long-column kernel's hot loop has no registers to spare: even values re-read from shared
// memory cost the long lists ~2% (measured).
template <bool kClampA, int kVar>
__global__ void __launch_bounds__(kListThreads, 2) prune_pairs_fine_kernel(const PruneArgs a) {
  constexpr bool kFine = true;
  extern __shared__ __align__(128) unsigned char smem[];
  // segmentation of this list, re-read from shared memory where it is used
  __shared__ int s_seg[2];
  __shared__ long long s_pstride;
  const int lane = threadIdx.x & 31;
  const TabAddr tp = load_tables_aligned(smem, a.g_exp, a.g_log, lane);
  if (kFine && threadIdx.x == 0) {
    // Short lists (fewer items than a.fine_items): finer sample segments, so that a stage of
    // a few hundred pairs still spreads over every SM. A pure function of the whole stage
    // list's length and n (not of this rank's slice), so a pair's bits do not depend on the
    // rank count; the part buffer holds nseg x pstride entries either way.
    int seg_len = a.seg_len, nseg = a.nseg;
    long long pstride = a.batch;
    const int all = a.off[a.u];
    const int all_chunks = (all + 31) / 32;
    while (all_chunks * nseg < a.fine_items && seg_len >= 2 * kMinSegLen && 2 * all <= pstride) {
      seg_len >>= 1;
      nseg = static_cast<int>((a.n + seg_len - 1) / seg_len);
      pstride >>= 1;
    }
    s_seg[0] = seg_len;
    s_seg[1] = nseg;
    s_pstride = pstride;
  }
  __syncthreads();
  const volatile int* vseg = s_seg;
  const volatile long long* vps = &s_pstride;
  cg::grid_group grid = cg::this_grid();
  const bool skip = (*a.err != kNoError);  // only skips work: every CTA still meets the barriers
  // this launch's share of the list: [kb, ke) — host-planned (k_end < 0: to the end of the
  // list), or this rank's slice of ceil(total / shard_world) entries planned here
  int kb = a.k_begin, ke = a.k_end >= 0 ? a.k_end : a.off[a.u];
  if (a.shard_world > 0) {
    const int tot = a.off[a.u];
    const int cnt = (tot + a.shard_world - 1) / a.shard_world;
    kb = min(tot, a.shard_rank * cnt);
    ke = min(tot, (a.shard_rank + 1) * cnt);
    if (cnt > a.shard_slot) {  // the host-side slot bound broke: ranks would overwrite each other's slots
      if (blockIdx.x == 0 && threadIdx.x == 0) atomicMin(a.err, err_key(0, kErrInternal, -1));
      ke = kb;
    }
  }
  const int total = ke - kb;
  const int nbatch = (total + a.batch - 1) / a.batch;
  for (int b = 0; b < nbatch; ++b) {
    if (b > 0) grid.sync();  // every chunk of batch b - 1 is finalised: the part slab is free
    const int base = kb + b * a.batch;
    const int m = min(a.batch, total - b * a.batch);
    const int chunks = (m + 31) / 32;
    int it = 0;
    if (lane == 0 && !skip) it = atomicAdd(&a.work[b], 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    while (!skip) {
      int nseg = kFine ? vseg[1] : a.nseg;
      if (it >= chunks * nseg) break;
      int chunk, seg;
      if (a.seg_major) {  // a sample window of every chunk at a time: column slices stay in L2
        seg = it / chunks;
        chunk = it - seg * chunks;
      } else {  // a chunk's segments back to back: its partial sums stay in L2
        chunk = it / nseg;
        seg = it - chunk * nseg;
      }
      const int kk = chunk * 32 + lane;
      if (kk < m) {
        int p, q;
        list_entry(a, base + kk, p, q);
        const int ci = a.act[p], cj = a.act[q];
        const double* wi = a.W + static_cast<int64_t>(ci) * a.ldw;
        const double* wj = a.W + static_cast<int64_t>(cj) * a.ldw;
        const int seg_len = kFine ? vseg[0] : a.seg_len;
        const int64_t t0 = static_cast<int64_t>(seg) * seg_len;  // multiple of 4: 32-byte aligned
        const int64_t t1 = lmin(a.n, t0 + seg_len);
        EdeAcc acc1, acc2;
        if (kVar == 4) {
          double2 xa = make_double2(0.0, 0.0), xb = xa, ya = xa, yb = xa;
          if (t0 + 3 < t1) {
            const double2* pi = reinterpret_cast<const double2*>(wi + t0);
            const double2* pj = reinterpret_cast<const double2*>(wj + t0);
            xa = __ldg(pi), xb = __ldg(pi + 1), ya = __ldg(pj), yb = __ldg(pj + 1);
          }
          double s1, bs1, s2, bs2;
          pair_scales(a.C, a.ldc, ci, cj, s1, bs1, s2, bs2);  // collinear pairs: zeros (flagged by predict)
          eval_segment_pre<kClampA>(wi, wj, t0, t1, s1, bs1, s2, bs2, acc1, acc2, tp, xa, xb, ya, yb);
        } else {
          double s1, bs1, s2, bs2;
          pair_scales(a.C, a.ldc, ci, cj, s1, bs1, s2, bs2);  // collinear pairs: zeros (flagged by predict)
          eval_segment<kClampA, kVar>(wi, wj, t0, t1, s1, bs1, s2, bs2, acc1, acc2, tp);
        }
        double2* dst = reinterpret_cast<double2*>(a.part + (static_cast<int64_t>(seg) * (kFine ? static_cast<int64_t>(*vps) : static_cast<int64_t>(a.batch)) + kk) * 4);
        __stcg(dst, make_double2(acc_lc(acc1), acc_pdf(acc1)));
        __stcg(dst + 1, make_double2(acc_lc(acc2), acc_pdf(acc2)));
      }
      fence_release_gpu();  // release this segment's partials before counting it (no L1 invalidation)
      __syncwarp();
      nseg = kFine ? vseg[1] : a.nseg;
      int last = 0, next = 0;
      if (lane == 0) {  // the segment count and the next item's fetch in one round trip
        last = (atomicAdd(&a.done[chunk], 1) == nseg - 1);
        next = atomicAdd(&a.work[b], 1);
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      it = __shfl_sync(0xffffffffu, next, 0);
      if (last) {
        fence_acquire_gpu();  // acquire the other segments' partials
        finalize_chunk_fine(a, a.part, base, m, chunk, lane, kb, nseg,
                       kFine ? static_cast<int64_t>(*vps) : static_cast<int64_t>(a.batch));
        if (lane == 0) a.done[chunk] = 0;  // ready for the next batch / launch
      }
    }
  }
}

// ---- scatter (multi-rank): every rank's results of the stage's list into Md / KN ----
__global__ void prune_scatter_kernel(const PruneArgs a, int world, int slot, int p2p_wait) {
  if (p2p_wait) {  // peer memory: every rank's entries of this stage must be in res first
    if (threadIdx.x == 0) p2p_wait_dev(a.peers);
    __syncthreads();
  }
  const int total = a.off[a.u];
  const int cnt = (total + world - 1) / world;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
    int p, q;
    list_entry(a, k, p, q);
    store_pair(a, p, q, a.res[(k / cnt) * slot + (k % cnt)]);
  }
}

// ---- bound: partial (or exact) k per row from the evaluated pairs ----
// pass 0 (after the probe): k* over the top rows' exact k; pass 1: alive rows' L (unused:
// the selection kernels compute L themselves); pass 2 (final): exact k of the top and alive
// rows, +inf else.
__global__ void __launch_bounds__(256) prune_bound_kernel(const PruneArgs a, int pass) {
  const int p = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= a.u) return;
  if (*a.err != kNoError) return;
  const int st = a.state_in[p];
  if (pass == 2 && st == 0) {
    if (lane == 0) a.k[p] = __longlong_as_double(static_cast<long long>(kInfBits));
    return;
  }
  if ((pass == 0 && st != 2) || (pass == 1 && st != 1)) return;
  const double* md = a.Md + static_cast<int64_t>(p) * a.u;
  // kreduce_kernel's lane-strided order: for a fully evaluated row this is its exact k bits
  double acc = 0.0;
#pragma unroll 4
  for (int q = lane; q < a.u; q += 32) {
    const double mi = md[q];
    if (q == p || !is_eval(mi)) continue;
    const double c = (mi < 0.0) ? mi : 0.0;
    acc = __dadd_rn(acc, __dmul_rn(c, c));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane != 0) return;
  if (pass == 2) {
    a.k[p] = acc;
  } else {
    a.L[p] = acc;
    if (st == 2) atomicMin(a.kstar, static_cast<unsigned long long>(__double_as_longlong(acc)));
  }
}

template <bool kClampA, int kVar, bool kFine = false>
int pairs_grid_for() {
  static DeviceCache gridc;
  const auto k = kFine ? prune_pairs_fine_kernel<kClampA, kVar> : prune_pairs_kernel<kClampA, kVar>;
  return gridc.get([k] {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kTableAlignedBytes);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kListThreads,
                                                  kTableAlignedBytes);
    return sms * (per > 0 ? per : 1);
  });
}

template <bool kClampA, int kVar, bool kFine = false>
cudaError_t launch_pairs_cfg(const PruneArgs& a, cudaStream_t s) {
  const int grid = pairs_grid_for<kClampA, kVar, kFine>();
  const auto k = kFine ? prune_pairs_fine_kernel<kClampA, kVar> : prune_pairs_kernel<kClampA, kVar>;
  PruneArgs args = a;
  void* params[] = {&args};
  // the grid barrier between batches needs every CTA resident: a failed cooperative launch
  // (e.g. fewer co-resident CTAs under a tool) must surface, not be skipped silently
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k),
                                     dim3(grid), dim3(kListThreads), params, kTableAlignedBytes, s);
}

}  // namespace

void launch_prune_predict(const PruneArgs& a, cudaStream_t s) {
  prune_predict_kernel<<<a.u, kPredThreads, 0, s>>>(a);
}

void launch_prune_top(const PruneArgs& a, int R, cudaStream_t s) {
  prune_top_kernel<<<1, kTopThreads, 0, s>>>(a, R < kMaxR ? R : kMaxR);
}

void launch_prune_select(const PruneArgs& a, int stage, int m, double beta, cudaStream_t s) {
  if (stage == kStageProbe) prune_probe_select_kernel<<<(a.u + 7) / 8, 256, 0, s>>>(a, m < kMaxT ? m : kMaxT);
  else {
    prune_rowl_kernel<<<a.u, kRowThreads, 0, s>>>(a);
    // the row's predictions cached in shared memory (u <= 24 576; larger rows re-read them)
    static DeviceCache attr;
    attr.get([] {
      cudaFuncSetAttribute(prune_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 24576 * 8);
      return 1;
    });
    const int cache = a.u <= 24576 ? 1 : 0;
    prune_select_kernel<<<a.u, kSelThreads, cache ? a.u * sizeof(double) : 0, s>>>(a, stage, m, beta, cache);
  }
}

void launch_prune_scan(const PruneArgs& a, cudaStream_t s) { prune_scan_kernel<<<1, 1024, 0, s>>>(a); }

namespace {
int fine_max_u() {
  static const int v = [] {  // PLG_FINE_MAX_U: the short-list kernel also for rounds up to this u
    const char* e = std::getenv("PLG_FINE_MAX_U");
    return e ? std::atoi(e) : 700;  // C3 -2%, C5 -0.3% (the long lists of large rounds keep the lean kernel)
  }();
  return v;
}
}  // namespace

// true when launch_prune_pairs takes the short-list kernel, whose sample segmentation (and
// with it each pair's bits) depends on the length of the list the pair is in
static bool prune_short_list_kernel(int u, int64_t n, int fine_items) {
  return n <= 90000 && fine_items > 0 && (n <= kFineMaxN || u <= fine_max_u());
}

cudaError_t launch_prune_pairs(const PruneArgs& a, cudaStream_t s) {
  static const int var = [] {  // PLG_LIST_VAR: load-pipeline variant (tuning knob)
    const char* v = std::getenv("PLG_LIST_VAR");
    return v ? std::atoi(v) : 0;
  }();
  if (a.n > 90000) return launch_pairs_cfg<true, 5>(a, s);
  if (prune_short_list_kernel(a.u, a.n, a.fine_items)) return launch_pairs_cfg<false, 5, true>(a, s);
  if (var == 1) return launch_pairs_cfg<false, 1>(a, s);
  if (var == 2) return launch_pairs_cfg<false, 2>(a, s);
  if (var == 4) return launch_pairs_cfg<false, 4>(a, s);
  if (var == 10) return launch_pairs_cfg<false, 0>(a, s);  // 128-bit loads (round-1 default)
  return launch_pairs_cfg<false, 5>(a, s);  // 256-bit loads: LDG.E.ENL2.256
}

void launch_prune_scatter(const PruneArgs& a, int world, int slot, cudaStream_t s, bool p2p_wait) {
  prune_scatter_kernel<<<148 * 4, 256, 0, s>>>(a, world, slot, p2p_wait ? 1 : 0);
}

void launch_prune_bound(const PruneArgs& a, int pass, cudaStream_t s) {
  prune_bound_kernel<<<(a.u + 7) / 8, 256, 0, s>>>(a, pass);
}


}  // namespace plg
