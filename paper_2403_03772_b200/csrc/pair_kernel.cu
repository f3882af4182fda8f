// pair_kernel.cu — the all-pairs residual-entropy kernel and its per-round companions.
//
// Replaces the reference's candidate_score inner loop (proj/src/ordering.cpp:78-99 →
// kernels.cpp:65-85,134-148): for every unordered pair {i, j} of active columns, both
// residual entropies E(i|j) and E(j|i) are evaluated once (the reference evaluates each
// twice, once per ordered pair). The pair's slopes and residual standard deviations come
// from the maintained Gram C (b = C_ij/C_jj, sd = sqrt(C_ii - C_ij b)), so the per-sample
// work is one residual, two exponentials and one log1p per direction.
//
// Work decomposition: a CTA owns one 32x32 tile of (i-block, j-block) positions and one
// sample segment. Each compute thread owns NI x 2 pairs x 2 directions (NI = 2: 256
// compute threads, 8 EDE per sample; NI = 1: 512 threads, 4 EDE) with per-thread
// left-to-right sums (the reduction order depends only on (u, n), never on the tile
// schedule or the GPU count). A dedicated producer warp stages 64-sample column chunks
// in shared memory with cp.async.bulk (one bulk copy per column chunk, mbarrier
// complete_tx) into a 3-stage ring; consumer warps release stages through per-stage
// "empty" mbarriers, so no CTA-wide barrier sits in the main loop.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "plg_async.cuh"
#include "plg_kernels.h"
#include "plg_math.cuh"
#include "plg_pair.cuh"

namespace plg {

namespace {

// Per-pair scales of both directions (plg_pair.cuh); zeros and the error key for an exactly
// collinear pair.
__device__ __forceinline__ void pair_params(const PairLaunch& a, int ci, int cj, double& s1, double& bs1,
                                            double& s2, double& bs2) {
  if (!pair_scales(a.C, a.ldc, ci, cj, s1, bs1, s2, bs2)) atomicMin(a.err, err_key(a.round, kErrPairCollinear, -1));
}

constexpr int kStages = 3;
constexpr int kStageDoubles = 2 * kBT * kCHS;
constexpr size_t kPairSmem = static_cast<size_t>(kTableBytes) + kStages * kStageDoubles * sizeof(double) +
                             2 * kStages * sizeof(uint64_t) + 2 * kBT * sizeof(int);

// Thread geometry: each compute thread owns NI i-positions x NJ j-positions of the 32x32
// tile (NQ = NI * NJ pairs, 2 NQ EDE per sample). kDedicated adds a producer warp; else the
// last compute warp also refills the ring.
template <int NI, int NJ, bool kDedicated>
struct PairCfg {
  static constexpr int NQ = NI * NJ;
  static constexpr int kCompute = kTilePairs / NQ;  // compute threads
  static constexpr int kWarps = kCompute / 32;
  static constexpr int kThreads = kCompute + (kDedicated ? 32 : 0);
  static constexpr int kIStride = kBT / NI;  // i positions ti + kIStride * x
  static constexpr int kJStride = kBT / NJ;  // j positions tj + kJStride * y
  static constexpr int kJGroups = kJStride / 8;  // warps along j (8 j-lanes per warp)
  static_assert(kWarps * 32 == kCompute && kJStride % 8 == 0, "geometry");
};

template <int NI, int NJ, bool kDedicated, bool kClampA>
__global__ void __launch_bounds__(PairCfg<NI, NJ, kDedicated>::kThreads, 1) pair_kernel(const PairLaunch a) {
  using Cfg = PairCfg<NI, NJ, kDedicated>;
  constexpr int NQ = Cfg::NQ;
  extern __shared__ __align__(128) unsigned char smem[];
  double* s_data = reinterpret_cast<double*>(smem + kTableBytes);
  uint64_t* s_full = reinterpret_cast<uint64_t*>(s_data + kStages * kStageDoubles);
  uint64_t* s_empty = s_full + kStages;
  int* s_col = reinterpret_cast<int*>(s_empty + kStages);
  __shared__ int s_abort;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int tl = blockIdx.x / a.nseg;        // tile within this launch
  const int seg = blockIdx.x - tl * a.nseg;  // sample segment
  int bi, bj;
  tile_decode(a.tile_begin + tl, a.nb, bi, bj);
  const bool diag = (bi == bj);

  if (tid == 0) s_abort = (*a.err != kNoError);
  if (tid < 2 * kBT) {
    const int p = (tid < kBT ? bi : bj) * kBT + (tid & (kBT - 1));
    s_col[tid] = (p < a.u) ? a.act[p] : -1;
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], Cfg::kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  load_tables(smem, a.g_exp, a.g_log);
  __syncthreads();
  if (s_abort) return;

  const int ncols = diag ? kBT : 2 * kBT;
  // Rows of columns past the active set are zero so they contribute exact zeros.
  for (int idx = tid; idx < kStages * ncols * kCHS; idx += Cfg::kThreads) {
    const int st = idx / (ncols * kCHS);
    const int row = (idx / kCHS) % ncols;
    if (s_col[row] < 0) s_data[st * kStageDoubles + row * kCHS + idx % kCHS] = 0.0;
  }
  const int64_t t_seg0 = static_cast<int64_t>(seg) * a.seg_len;
  const int64_t t_seg1 = lmin(a.n, t_seg0 + a.seg_len);
  const int nch = static_cast<int>((t_seg1 - t_seg0 + kCH - 1) / kCH);
  int nvalid = 0;
  for (int r = 0; r < ncols; ++r) nvalid += (s_col[r] >= 0);
  __syncthreads();  // zero-fill visible before the first chunk is consumed

  auto issue = [&](int c) {  // one warp: stage chunk c into ring slot c % kStages
    const int st = c % kStages;
    const int64_t t0 = t_seg0 + static_cast<int64_t>(c) * kCH;
    const int len = static_cast<int>(lmin(kCH, t_seg1 - t0));
    const uint32_t bytes = static_cast<uint32_t>(((len + 1) & ~1) * sizeof(double));
    if (lane == 0) mbar_expect_tx(&s_full[st], bytes * nvalid);
    __syncwarp();
    for (int r = lane; r < ncols; r += 32) {
      const int col = s_col[r];
      if (col >= 0)
        bulk_g2s(s_data + st * kStageDoubles + r * kCHS, a.W + static_cast<int64_t>(col) * a.ldw + t0, bytes,
                 &s_full[st]);
    }
  };
  const int producer = kDedicated ? Cfg::kWarps : Cfg::kWarps - 1;
  if (kDedicated && warp == producer) {  // ---- dedicated producer warp ----
    for (int c = 0; c < nch; ++c) {
      if (c >= kStages) mbar_wait(&s_empty[c % kStages], ((c / kStages) - 1) & 1);
      issue(c);
    }
    return;
  }
  if (!kDedicated && warp == producer)
    for (int c = 0; c < kStages && c < nch; ++c) issue(c);

  // ---- compute warps: pairs (ti + kIStride*x, tj + kJStride*y) ----
  const int ti = (warp / Cfg::kJGroups) * 4 + (lane >> 3);
  const int tj = (warp % Cfg::kJGroups) * 8 + (lane & 7);
  double s1[NQ], bs1[NQ], s2[NQ], bs2[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int pi = ti + Cfg::kIStride * (q / NJ);
    const int pj = tj + Cfg::kJStride * (q % NJ);
    const int ci = s_col[pi];
    const int cj = s_col[diag ? pj : kBT + pj];
    const bool valid = (ci >= 0) && (cj >= 0) && (!diag || pi < pj);
    s1[q] = bs1[q] = s2[q] = bs2[q] = 0.0;
    if (valid) pair_params(a, ci, cj, s1[q], bs1[q], s2[q], bs2[q]);
  }
  EdeAcc acc[2 * NQ];  // [q] direction i|j, [NQ + q] direction j|i
  const TabPtr tp = table_ptrs(smem, lane);
  const int jrow = diag ? 0 : kBT;

  for (int c = 0; c < nch; ++c) {
    const int st = c % kStages;
    if (!kDedicated && warp == producer && c >= 1 && c - 1 + kStages < nch) {
      // refill the slot chunk c-1 used once every warp has released it
      mbar_wait(&s_empty[(c - 1) % kStages], ((c - 1) / kStages) & 1);
      issue(c - 1 + kStages);
    }
    mbar_wait(&s_full[st], (c / kStages) & 1);
    const double* base = s_data + st * kStageDoubles;
    const double* xip[NI];
    const double* xjp[NJ];
#pragma unroll
    for (int x = 0; x < NI; ++x) xip[x] = base + (ti + Cfg::kIStride * x) * kCHS;
#pragma unroll
    for (int y = 0; y < NJ; ++y) xjp[y] = base + (jrow + tj + Cfg::kJStride * y) * kCHS;
    const int len = static_cast<int>(lmin(kCH, t_seg1 - (t_seg0 + static_cast<int64_t>(c) * kCH)));
#pragma unroll 1
    for (int t = 0; t < len; ++t) {
      double xi[NI], xj[NJ];
#pragma unroll
      for (int x = 0; x < NI; ++x) xi[x] = xip[x][t];
#pragma unroll
      for (int y = 0; y < NJ; ++y) xj[y] = xjp[y][t];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const double x = xi[q / NJ];
        const double y = xj[q % NJ];
        const double u1 = fma(y, -bs1[q], x * s1[q]);  // (x_i - b_ij x_j) / sd_ij
        const double u2 = fma(x, -bs2[q], y * s2[q]);  // (x_j - b_ji x_i) / sd_ji
        ede_accumulate<kClampA>(u1, acc[q], tp);
        ede_accumulate<kClampA>(u2, acc[NQ + q], tp);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&s_empty[st]);
  }

#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int slot = (ti + Cfg::kIStride * (q / NJ)) * kBT + tj + Cfg::kJStride * (q % NJ);
    double2* dst = reinterpret_cast<double2*>(
        a.part + ((static_cast<int64_t>(tl) * a.nseg + seg) * kTilePairs + slot) * 4);
    dst[0] = make_double2(acc_lc(acc[q]), acc_pdf(acc[q]));
    dst[1] = make_double2(acc_lc(acc[NQ + q]), acc_pdf(acc[NQ + q]));
  }
}

// Sum the segment partials (ascending) and form both residual entropies of each pair:
// epack[tile][0][x][y] = E(a_x | b_y), epack[tile][1][y][x] = E(b_y | a_x).
__global__ void finalize_kernel(const PairLaunch a) {
  if (*a.err != kNoError) return;
  const int tl = blockIdx.x;
  const int slot = blockIdx.y * blockDim.x + threadIdx.x;
  const int x = slot / kBT, y = slot % kBT;
  int bi, bj;
  tile_decode(a.tile_begin + tl, a.nb, bi, bj);
  const bool valid = (bi * kBT + x < a.u) && (bj * kBT + y < a.u) && (bi != bj || x < y);
  double e1 = 0.0, e2 = 0.0;
  if (valid) {
    double l1 = 0.0, p1 = 0.0, l2 = 0.0, p2 = 0.0;
    const double* src = a.part + (static_cast<int64_t>(tl) * a.nseg * kTilePairs + slot) * 4;
    for (int s = 0; s < a.nseg; ++s) {
      const double2 v1 = reinterpret_cast<const double2*>(src)[0];
      const double2 v2 = reinterpret_cast<const double2*>(src)[1];
      l1 += v1.x;
      p1 += v1.y;
      l2 += v2.x;
      p2 += v2.y;
      src += static_cast<int64_t>(kTilePairs) * 4;
    }
    const double inv_n = 1.0 / static_cast<double>(a.n);
    e1 = entropy_from_sums(l1, p1, inv_n);
    e2 = entropy_from_sums(l2, p2, inv_n);
  }
  double* tile = a.epack + static_cast<int64_t>(a.tile_begin + tl) * 2 * kTilePairs;
  if (a.peers.n > 0) {  // every rank's copy of the table (peer memory), then p2p_signal
    peer_store(a.peers, &tile[x * kBT + y], e1);
    peer_store(a.peers, &tile[kTilePairs + y * kBT + x], e2);  // published by p2p_signal after this kernel
    return;
  }
  tile[x * kBT + y] = e1;
  tile[kTilePairs + y * kBT + x] = e2;
}

// (p, q), p < q < u, of the p-major pair index.
__device__ __forceinline__ void pair_decode(int pair, int u, int& p, int& q) {
  int rem = pair;
  p = 0;
  while (rem >= u - 1 - p) {
    rem -= u - 1 - p;
    ++p;
  }
  q = p + 1 + rem;
}

template <bool kClampA>
__global__ void __launch_bounds__(kSmallThreads) pair_small_kernel(const PairLaunch a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int s_abort;
  if (threadIdx.x == 0) s_abort = (*a.err != kNoError);
  load_tables(smem, a.g_exp, a.g_log);
  __syncthreads();
  if (s_abort) return;
  const int npairs = a.u * (a.u - 1) / 2;
  const int pair = blockIdx.x * kSmallThreads + threadIdx.x;
  if (pair >= npairs) return;
  const int seg = blockIdx.y;
  int p, q;
  pair_decode(pair, a.u, p, q);
  double s1, bs1, s2, bs2;
  pair_params(a, a.act[p], a.act[q], s1, bs1, s2, bs2);
  const double* wi = a.W + static_cast<int64_t>(a.act[p]) * a.ldw;
  const double* wj = a.W + static_cast<int64_t>(a.act[q]) * a.ldw;
  const TabPtr tp = table_ptrs(smem, threadIdx.x & 31);
  EdeAcc acc1, acc2;
  const int64_t t0 = static_cast<int64_t>(seg) * a.seg_len;  // multiple of 16: 32-byte aligned
  const int64_t t1 = lmin(a.n, t0 + a.seg_len);
  int64_t t = t0;
  auto ede2 = [&](double x, double y) {
    ede_accumulate<kClampA>(fma(y, -bs1, x * s1), acc1, tp);
    ede_accumulate<kClampA>(fma(x, -bs2, y * s2), acc2, tp);
  };
  // 4 samples per step with 256-bit loads, the next step's loads issued before this step's math
  const int nstep = static_cast<int>((t1 - t0) >> 2);
  if (nstep > 0) {
    const double* pi = wi + t0;
    const double* pj = wj + t0;
    double4 x = ldg256(pi), y = ldg256(pj);
#pragma unroll 1
    for (int i = 1; i <= nstep; ++i) {
      const double4 cx = x, cy = y;
      pi += 4;
      pj += 4;
      if (i < nstep) x = ldg256(pi), y = ldg256(pj);
      ede2(cx.x, cy.x);
      ede2(cx.y, cy.y);
      ede2(cx.z, cy.z);
      ede2(cx.w, cy.w);
    }
    t += 4 * static_cast<int64_t>(nstep);
  }
  for (; t < t1; ++t) ede2(wi[t], wj[t]);
  double2* dst = reinterpret_cast<double2*>(a.part + (static_cast<int64_t>(seg) * npairs + pair) * 4);
  dst[0] = make_double2(acc_lc(acc1), acc_pdf(acc1));
  dst[1] = make_double2(acc_lc(acc2), acc_pdf(acc2));
}

__global__ void finalize_small_kernel(const PairLaunch a) {
  if (*a.err != kNoError) return;
  const int npairs = a.u * (a.u - 1) / 2;
  const int pair = blockIdx.x * blockDim.x + threadIdx.x;
  if (pair >= npairs) return;
  int p, q;
  pair_decode(pair, a.u, p, q);
  double l1 = 0.0, p1 = 0.0, l2 = 0.0, p2 = 0.0;
  const double* src = a.part + static_cast<int64_t>(pair) * 4;
  for (int s = 0; s < a.nseg; ++s) {
    const double2 v1 = reinterpret_cast<const double2*>(src)[0];
    const double2 v2 = reinterpret_cast<const double2*>(src)[1];
    l1 += v1.x;
    p1 += v1.y;
    l2 += v2.x;
    p2 += v2.y;
    src += static_cast<int64_t>(npairs) * 4;
  }
  const double inv_n = 1.0 / static_cast<double>(a.n);
  const int bi = p / kBT, x = p % kBT, bj = q / kBT, y = q % kBT;
  double* tile = a.epack + static_cast<int64_t>(bi * a.nb - (bi * (bi - 1)) / 2 + (bj - bi)) * 2 * kTilePairs;
  tile[x * kBT + y] = entropy_from_sums(l1, p1, inv_n);
  tile[kTilePairs + y * kBT + x] = entropy_from_sums(l2, p2, inv_n);
}

constexpr int kColentThreads = 256;

// H_p = entropy_approx(standardised column) (ordering.cpp:65; kernels.cpp:123-132).
__global__ void __launch_bounds__(kColentThreads)
    colent_kernel(const double* W, int64_t ldw, int64_t n, const double* C, int64_t ldc,
                  const int* act, int u, double* H, const double* g_exp, const double2* g_log,
                  const int* nz, const int* col_var, int round, unsigned long long* err) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double s_red[2][kColentThreads / 32];
  if (*err != kNoError) return;
  load_tables(smem, g_exp, g_log);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const TabPtr tp = table_ptrs(smem, lane);
  for (int p = blockIdx.x; p < u; p += gridDim.x) {
    const int col = act[p];
    const double ccc = C[static_cast<int64_t>(col) * ldc + col];
    if (round > 0 && threadIdx.x == 0 && (nz[col] != round || !(ccc > 0.0)))
      atomicMin(err, err_key(round, kErrColZeroVar, col_var[col]));  // ordering.cpp:56-62
    const double inv_sd = 1.0 / sqrt(ccc);
    const double* w = W + static_cast<int64_t>(col) * ldw;
    EdeAcc acc;
    const double su = inv_sd * kUScale;
    for (int64_t t = threadIdx.x; t < n; t += kColentThreads) ede_accumulate<true>(w[t] * su, acc, tp);
    double lc = acc_lc(acc), pd = acc_pdf(acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lc += __shfl_xor_sync(0xffffffffu, lc, o);
      pd += __shfl_xor_sync(0xffffffffu, pd, o);
    }
    if (lane == 0) {
      s_red[0][warp] = lc;
      s_red[1][warp] = pd;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double l = 0.0, q = 0.0;
      for (int w2 = 0; w2 < kColentThreads / 32; ++w2) {
        l += s_red[0][w2];
        q += s_red[1][w2];
      }
      H[p] = entropy_from_sums(l, q, 1.0 / static_cast<double>(n));
    }
    __syncthreads();
  }
}

// Residualisation fused with the next round's column entropies: w_r <- w_r - (C_rm / C_mm) w_m
// in place (multiply then subtract, as residual_into) and, from the new values already in registers,
// the entropy sums of w_r / sqrt(C_rr) (C after the rank-1 update) per sample chunk:
// hpart[(r * nch + c) * 2] = {sum lc, sum pdf}. hfin_kernel adds the chunks in ascending
// order next round. Persistent CTAs so the tables are staged once per CTA, not per column.
constexpr int kResidThreads = 256;
// One warp per (column, chunk) item: lane-strided double2 pairs, a warp shuffle reduction, no
// block barrier; items are taken warp-strided over the persistent grid.
__global__ void __launch_bounds__(kResidThreads)
    resid_ent_kernel(double* W, int64_t ldw, int64_t n, const double* C, int64_t ldc, const int* act_nxt,
                     int ur, const RoundState* rs, int* nz, int tag, const unsigned long long* err,
                     int64_t chunk, int nch, double* hpart, const double* g_exp, const double2* g_log,
                     int c_updated) {
  extern __shared__ __align__(128) unsigned char smem[];
  if (*err != kNoError) return;
  load_tables(smem, g_exp, g_log);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const TabPtr tp = table_ptrs(smem, lane);
  const int m = rs->chosen_col;
  const double cmm = C[static_cast<int64_t>(m) * ldc + m];
  const double2* wm = reinterpret_cast<const double2*>(W + static_cast<int64_t>(m) * ldw);
  const int items = ur * nch;
  const int warps = gridDim.x * (kResidThreads / 32);
  for (int it = blockIdx.x * (kResidThreads / 32) + (threadIdx.x >> 5); it < items; it += warps) {
    const int pos = it / nch, c = it - pos * nch;
    const int r = act_nxt[pos];
    const double beta = C[static_cast<int64_t>(r) * ldc + m] / cmm;
    const double crr = c_updated ? C[static_cast<int64_t>(r) * ldc + r]
                                 : gram_update_entry(C[static_cast<int64_t>(r) * ldc + r], C[static_cast<int64_t>(r) * ldc + m],
                                                     C[static_cast<int64_t>(m) * ldc + r], cmm);
    const double su = kUScale / sqrt(crr);
    double2* wr = reinterpret_cast<double2*>(W + static_cast<int64_t>(r) * ldw);
    const int64_t t0 = c * chunk, t1 = lmin(n, t0 + chunk);  // samples; chunk is even
    EdeAcc acc;
    bool any = false;
    // loads of the next step issued before this step's element math (latency-bound otherwise)
    int64_t t = t0 + 2 * lane;
    double2 xn = make_double2(0.0, 0.0), yn = xn;
    if (t < t1) xn = wr[t >> 1], yn = wm[t >> 1];
    for (; t < t1; t += 64) {
      const double2 x = xn, y = yn;
      if (t + 64 < t1) xn = wr[(t + 64) >> 1], yn = wm[(t + 64) >> 1];
      const double2 o = make_double2(__dsub_rn(x.x, __dmul_rn(beta, y.x)), __dsub_rn(x.y, __dmul_rn(beta, y.y)));
      wr[t >> 1] = o;
      any |= (o.x != 0.0) | (o.y != 0.0);
      ede_accumulate<true>(o.x * su, acc, tp);
      if (t + 1 < t1) ede_accumulate<true>(o.y * su, acc, tp);
    }
    if (__any_sync(0xffffffffu, any) && lane == 0) nz[r] = tag;
    double lc = acc_lc(acc), pd = acc_pdf(acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lc += __shfl_xor_sync(0xffffffffu, lc, o);
      pd += __shfl_xor_sync(0xffffffffu, pd, o);
    }
    if (lane == 0) {
      hpart[static_cast<int64_t>(it) * 2] = lc;
      hpart[static_cast<int64_t>(it) * 2 + 1] = pd;
    }
  }
}

// H[p] from resid_ent_kernel's chunk sums (ascending chunks), plus build_cache's
// ZeroVariance(col) check of the round (ordering.cpp:56-62), as colent_kernel does.
__global__ void hfin_kernel(const double* hpart, int nch, int64_t n, const double* C, int64_t ldc, const int* act,
                            int u, double* H, const int* nz, const int* col_var, int round,
                            unsigned long long* err) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= u) return;
  const int col = act[p];
  const double ccc = C[static_cast<int64_t>(col) * ldc + col];
  if (nz[col] != round || !(ccc > 0.0)) atomicMin(err, err_key(round, kErrColZeroVar, col_var[col]));
  double l = 0.0, q = 0.0;
  for (int c = 0; c < nch; ++c) {
    l += hpart[(static_cast<int64_t>(p) * nch + c) * 2];
    q += hpart[(static_cast<int64_t>(p) * nch + c) * 2 + 1];
  }
  H[p] = entropy_from_sums(l, q, 1.0 / static_cast<double>(n));
}

// entropy_approx(u * scale) of one vector (kernels.cpp:123-148), fixed-shape reduction.
__global__ void __launch_bounds__(kColentThreads)
    entropy_vec_kernel(const double* u, int64_t n, double scale, double* out, const double* g_exp,
                       const double2* g_log) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double s_red[2][kColentThreads / 32];
  load_tables(smem, g_exp, g_log);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const TabPtr tp = table_ptrs(smem, lane);
  EdeAcc acc;
  const double su = scale * kUScale;
  for (int64_t t = threadIdx.x; t < n; t += kColentThreads) ede_accumulate<true>(u[t] * su, acc, tp);
  double lc = acc_lc(acc), pd = acc_pdf(acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lc += __shfl_xor_sync(0xffffffffu, lc, o);
    pd += __shfl_xor_sync(0xffffffffu, pd, o);
  }
  if (lane == 0) {
    s_red[0][warp] = lc;
    s_red[1][warp] = pd;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double l = 0.0, q = 0.0;
    for (int w2 = 0; w2 < kColentThreads / 32; ++w2) {
      l += s_red[0][w2];
      q += s_red[1][w2];
    }
    *out = entropy_from_sums(l, q, 1.0 / static_cast<double>(n));
  }
}

__global__ void math_probe_kernel(const double* u, int64_t n, double* out, const double* g_exp,
                                  const double2* g_log) {
  extern __shared__ __align__(128) unsigned char smem[];
  load_tables(smem, g_exp, g_log);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const TabPtr tp = table_ptrs(smem, lane);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = u[i];
    EdeAcc acc;
    ede_accumulate<true>(v * kUScale, acc, tp);
    const double lc = acc_lc(acc), pd = acc_pdf(acc);
    const double a = fabs(v);
    out[4 * i + 0] = lc;
    out[4 * i + 1] = pd;
    out[4 * i + 2] = a + (log1p(exp(-2.0 * a)) - kLn2);  // libdevice, kernels.cpp:22-23
    out[4 * i + 3] = v * exp(-0.5 * (v * v));            // kernels.cpp:24
  }
}

template <int NI, int NJ, bool kDedicated, bool kClampA>
void launch_pair_cfg(const PairLaunch& a, cudaStream_t s) {
  static DeviceCache attr;
  attr.get([] {
    cudaFuncSetAttribute(pair_kernel<NI, NJ, kDedicated, kClampA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kPairSmem));
    return 1;
  });
  pair_kernel<NI, NJ, kDedicated, kClampA>
      <<<a.ntiles * a.nseg, PairCfg<NI, NJ, kDedicated>::kThreads, kPairSmem, s>>>(a);
}

}  // namespace

void launch_pair(const PairLaunch& a, cudaStream_t s) {
  // |u| <= sqrt(n) for a normalised residual; exp(-2|u|)'s scaling needs its clamp only past
  // |u| ~ 350 (plg_math.cuh).
  const bool clamp = a.n > 90000;
  // PLG_PAIR_GEOM selects the thread geometry (tuning knob): "22d" (default) = 2x2 pairs per
  // thread, 256 threads + a producer warp (measured 1-2% faster); "12" = 1x2 pairs, 512
  // threads, in-warp producer.
  static const bool g22 = [] {
    const char* v = std::getenv("PLG_PAIR_GEOM");
    return !(v && !strcmp(v, "12"));
  }();
  if (g22) {
    if (clamp) launch_pair_cfg<2, 2, true, true>(a, s);
    else launch_pair_cfg<2, 2, true, false>(a, s);
  } else {
    if (clamp) launch_pair_cfg<1, 2, false, true>(a, s);
    else launch_pair_cfg<1, 2, false, false>(a, s);
  }
}

void launch_finalize(const PairLaunch& a, cudaStream_t s) {
  finalize_kernel<<<dim3(a.ntiles, kTilePairs / 256), 256, 0, s>>>(a);
}

namespace {
template <bool kClampA>
void launch_pair_small_cfg(const PairLaunch& a, cudaStream_t s) {
  static DeviceCache attr;
  attr.get([] {
    cudaFuncSetAttribute(pair_small_kernel<kClampA>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTableBytes);
    return 1;
  });
  const int npairs = a.u * (a.u - 1) / 2;
  pair_small_kernel<kClampA>
      <<<dim3((npairs + kSmallThreads - 1) / kSmallThreads, a.nseg), kSmallThreads, kTableBytes, s>>>(a);
}
}  // namespace

void launch_pair_small(const PairLaunch& a, cudaStream_t s) {
  if (a.n > 90000) launch_pair_small_cfg<true>(a, s);
  else launch_pair_small_cfg<false>(a, s);
}

void launch_finalize_small(const PairLaunch& a, cudaStream_t s) {
  const int npairs = a.u * (a.u - 1) / 2;
  finalize_small_kernel<<<(npairs + 255) / 256, 256, 0, s>>>(a);
}

void launch_colent(const double* W, int64_t ldw, int64_t n, const double* C, int64_t ldc,
                   const int* act, int u, double* H, const double* g_exp, const double2* g_log,
                   const int* nz, const int* col_var, int round, unsigned long long* err,
                   cudaStream_t s) {
  static DeviceCache attr;
  attr.get([] {
    cudaFuncSetAttribute(colent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTableBytes);
    return 1;
  });
  const int grid = u < 4 * 148 ? u : 4 * 148;
  colent_kernel<<<grid, kColentThreads, kTableBytes, s>>>(W, ldw, n, C, ldc, act, u, H, g_exp,
                                                          g_log, nz, col_var, round, err);
}

int resid_chunks(int64_t n) { return static_cast<int>((n + kResidChunk - 1) / kResidChunk); }

void launch_resid_ent(double* W, int64_t ldw, int64_t n, const double* C, int64_t ldc, const int* act_nxt, int ur,
                      const RoundState* rs, int* nz, int tag, const unsigned long long* err, double* hpart,
                      const double* g_exp, const double2* g_log, cudaStream_t s, bool C_updated) {
  static DeviceCache gridc;
  const int grid = gridc.get([] {
    cudaFuncSetAttribute(resid_ent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTableBytes);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, resid_ent_kernel, kResidThreads, kTableBytes);
    return sms * (per > 0 ? per : 1);
  });
  const int nch = resid_chunks(n);
  const int need = (ur * nch + kResidThreads / 32 - 1) / (kResidThreads / 32);
  const int g = need < grid ? need : grid;
  resid_ent_kernel<<<g, kResidThreads, kTableBytes, s>>>(W, ldw, n, C, ldc, act_nxt, ur, rs, nz, tag, err,
                                                        kResidChunk, nch, hpart, g_exp, g_log, C_updated ? 1 : 0);
}

void launch_hfin(const double* hpart, int64_t n, const double* C, int64_t ldc, const int* act, int u, double* H,
                 const int* nz, const int* col_var, int round, unsigned long long* err, cudaStream_t s) {
  hfin_kernel<<<(u + 127) / 128, 128, 0, s>>>(hpart, resid_chunks(n), n, C, ldc, act, u, H, nz, col_var, round,
                                              err);
}

void launch_entropy_vec(const double* u, int64_t n, double scale, double* out, const double* g_exp,
                        const double2* g_log, cudaStream_t s) {
  static DeviceCache attr;
  attr.get([] {
    cudaFuncSetAttribute(entropy_vec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTableBytes);
    return 1;
  });
  entropy_vec_kernel<<<1, kColentThreads, kTableBytes, s>>>(u, n, scale, out, g_exp, g_log);
}

void launch_math_probe(const double* u, int64_t n, double* out, const double* g_exp,
                       const double2* g_log, cudaStream_t s) {
  static DeviceCache attr;
  attr.get([] {
    cudaFuncSetAttribute(math_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kTableBytes);
    return 1;
  });
  int grid = static_cast<int>((n + 255) / 256);
  if (grid > 1184) grid = 1184;
  if (grid < 1) grid = 1;
  math_probe_kernel<<<grid, 256, kTableBytes, s>>>(u, n, out, g_exp, g_log);
}

}  // namespace plg
