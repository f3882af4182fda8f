// round_kernels.cu — the O(u n) and O(u^2) kernels around the pair kernel:
// validation + standardisation, the one-off FP64 Gram, the k reduction, the lowest-index
// argmin with active-list compaction, the rank-1 Gram update and the in-place
// residualisation (reference proj/src/ordering.cpp:47-70,101-162,178-244,
// proj/src/kernels.cpp:44-121, proj/src/types.cpp:21-47).
#include <cuda_runtime.h>

#include "plg_kernels.h"

namespace plg {

namespace {

constexpr int kSeqChunk = 1024;  // per-warp staging for the left-to-right sums

// Left-to-right sum of f(x_t) by lane 0 of a warp (the reference's summation order,
// kernels.cpp:44-57), with the column staged through shared memory by all lanes.
// Explicit _rn intrinsics keep nvcc from contracting into FMAs (-ffp-contract=off).
template <typename F>
__device__ double warp_seq_sum(const double* x, int64_t n, double* buf, F f) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int64_t t0 = 0; t0 < n; t0 += kSeqChunk) {
    const int len = static_cast<int>(lmin(kSeqChunk, n - t0));
    __syncwarp();
    for (int i = lane; i < len; i += 32) buf[i] = x[t0 + i];
    __syncwarp();
    if (lane == 0)
      for (int i = 0; i < len; ++i) s = __dadd_rn(s, f(buf[i]));
  }
  return __shfl_sync(0xffffffffu, s, 0);
}

constexpr int kStdWarps = 4;

__global__ void __launch_bounds__(32 * kStdWarps)
    standardize_kernel(const double* X, int64_t ldx, int64_t n, const int* col_map, int ncol,
                       double* W, int64_t ldw, int* stat, double* msd, int check_finite) {
  __shared__ double buf[kStdWarps][kSeqChunk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * kStdWarps + warp;
  if (c >= ncol) return;
  const double* x = X + static_cast<int64_t>(col_map ? col_map[c] : c) * ldx;
  int first_bad = -1;
  if (check_finite) {  // types.cpp:27-35: first non-finite row of this column
    int bad = 0x7fffffff;
    for (int64_t t = lane; t < n; t += 32)
      if (!isfinite(x[t])) {
        bad = static_cast<int>(t);
        break;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    first_bad = (bad == 0x7fffffff) ? -1 : bad;
  }
  const double dn = static_cast<double>(n);
  const double m = warp_seq_sum(x, n, buf[warp], [](double v) { return v; }) / dn;  // mean()
  const double var =
      warp_seq_sum(x, n, buf[warp], [m](double v) {
        const double dv = v - m;
        return __dmul_rn(dv, dv);
      }) / dn;  // variance_pop_given_mean()
  if (lane == 0) {
    stat[2 * c] = first_bad;
    stat[2 * c + 1] = (var == 0.0);
  }
  const double sd = sqrt(var);  // std_pop()
  if (msd && lane == 0) {
    msd[2 * c] = m;
    msd[2 * c + 1] = sd;
  }
  double* w = W + static_cast<int64_t>(c) * ldw;
  for (int64_t t = lane; t < ldw; t += 32) w[t] = (t < n && sd != 0.0) ? (x[t] - m) / sd : 0.0;
}

// C = W^T W / n, 64x64 output tiles on the upper triangle, mirrored (bit-symmetric).
constexpr int kGT = 64, kGK = 16;
__global__ void __launch_bounds__(256) gram_kernel(const double* W, int64_t ldw, int64_t n, int ncol,
                                                   double* C, int64_t ldc, int ntb, int64_t chunk,
                                                   double* scratch) {
  __shared__ double As[kGK][kGT + 2];
  __shared__ double Bs[kGK][kGT + 2];
  int bi, bj;
  tile_decode(blockIdx.x, ntb, bi, bj);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  const int64_t tb = blockIdx.y * chunk;
  const int64_t te = lmin(n, tb + chunk);
  for (int64_t t0 = tb; t0 < te; t0 += kGK) {
    for (int e = threadIdx.x; e < kGK * kGT; e += 256) {
      const int tt = e % kGK, cc = e / kGK;
      const int ca = bi * kGT + cc, cb = bj * kGT + cc;
      const int64_t t = t0 + tt;
      As[tt][cc] = (ca < ncol && t < te) ? W[static_cast<int64_t>(ca) * ldw + t] : 0.0;
      Bs[tt][cc] = (cb < ncol && t < te) ? W[static_cast<int64_t>(cb) * ldw + t] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int tt = 0; tt < kGK; ++tt) {
      double av[4], bv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        av[r] = As[tt][ty * 4 + r];
        bv[r] = Bs[tt][tx * 4 + r];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int s = 0; s < 4; ++s) acc[r][s] = fma(av[r], bv[s], acc[r][s]);
    }
    __syncthreads();
  }
  if (gridDim.y > 1) {  // partial tile of this sample chunk
    double* dst = scratch + (static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x) * kGT * kGT;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int s = 0; s < 4; ++s) dst[(ty * 4 + r) * kGT + tx * 4 + s] = acc[r][s];
    return;
  }
  const double dn = static_cast<double>(n);
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int i = bi * kGT + ty * 4 + r, j = bj * kGT + tx * 4 + s;
      if (i < ncol && j < ncol) {
        const double v = acc[r][s] / dn;
        C[static_cast<int64_t>(i) * ldc + j] = v;
        C[static_cast<int64_t>(j) * ldc + i] = v;
      }
    }
}

// Sum the chunk partials in ascending chunk order and mirror (bit-symmetric C).
__global__ void gram_reduce_kernel(const double* scratch, int ntiles, int nchunk, int ntb, int64_t n,
                                   int ncol, double* C, int64_t ldc) {
  int bi, bj;
  tile_decode(blockIdx.x, ntb, bi, bj);
  const double dn = static_cast<double>(n);
  for (int e = threadIdx.x; e < kGT * kGT; e += blockDim.x) {
    const int r = e / kGT, s = e % kGT;
    const int i = bi * kGT + r, j = bj * kGT + s;
    if (i >= ncol || j >= ncol) continue;
    double v = 0.0;
    for (int c = 0; c < nchunk; ++c) v += scratch[(static_cast<int64_t>(c) * ntiles + blockIdx.x) * kGT * kGT + e];
    v /= dn;
    C[static_cast<int64_t>(i) * ldc + j] = v;
    C[static_cast<int64_t>(j) * ldc + i] = v;
  }
}

__device__ __forceinline__ int tile_index(int bi, int bj, int nb) {
  return bi * nb - (bi * (bi - 1)) / 2 + (bj - bi);
}

// Warp per candidate position p; lanes stride q, fixed xor-tree reduction. errs[0..world)
// are the ranks' error keys gathered with the entropy tiles (a pair error is seen only by
// the rank that owns the tile): every rank adopts the smallest, so all report the same.
__global__ void kreduce_kernel(const double* epack, const double* H, int u, int nb, double* k,
                               unsigned long long* err, const unsigned long long* errs, int world,
                               const int* act, double* KN, int d) {
  unsigned long long key = *err;
  for (int r = 0; r < world; ++r) key = min(key, errs[r]);
  if (key != kNoError) {
    if (threadIdx.x == 0) atomicMin(err, key);
    return;
  }
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= u) return;
  const int bp = p / kBT, xp = p % kBT;
  const double hp = H[p];
  double* kn = KN ? KN + static_cast<int64_t>(act[p]) * d : nullptr;
  double acc = 0.0;
  for (int q = lane; q < u; q += 32) {
    if (q == p) continue;
    const int bq = q / kBT, xq = q % kBT;
    double e_pq, e_qp;
    if (bp < bq || (bp == bq && xp < xq)) {
      const double* tile = epack + static_cast<int64_t>(tile_index(bp, bq, nb)) * 2 * kTilePairs;
      e_pq = tile[xp * kBT + xq];
      e_qp = tile[kTilePairs + xq * kBT + xp];
    } else {
      const double* tile = epack + static_cast<int64_t>(tile_index(bq, bp, nb)) * 2 * kTilePairs;
      e_pq = tile[kTilePairs + xp * kBT + xq];
      e_qp = tile[xq * kBT + xp];
    }
    // ordering.cpp:93-96: mi = (H_q + E(p|q)) - (H_p + E(q|p)); k += min(0, mi)^2
    const double mi = (H[q] + e_pq) - (hp + e_qp);
    const double c = (mi < 0.0) ? mi : 0.0;
    acc = __dadd_rn(acc, __dmul_rn(c, c));
    if (kn) kn[act[q]] = __dmul_rn(c, c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) k[p] = acc;
}

constexpr int kCommitThreads = 1024;

// ordering.cpp:154-160 argmax of -k with strict '>' over ascending candidates == argmin of
// k with the lowest position on ties. Then order bookkeeping and active-list compaction.
__global__ void __launch_bounds__(kCommitThreads)
    commit_kernel(const double* k, const int* act_cur, int* act_nxt, int u, const int* col_var,
                  int* order, int round, double* scores, RoundState* rs,
                  const unsigned long long* err, double* round_k, const double* lb, double* round_second) {
  __shared__ double sk[kCommitThreads];
  __shared__ int sp[kCommitThreads];
  __shared__ double s2[kCommitThreads];
  if (*err != kNoError) return;
  double best = 0.0;
  int bp = -1;
  for (int p = threadIdx.x; p < u; p += kCommitThreads) {
    const double v = k[p];
    if (bp < 0 || v < best) {
      best = v;
      bp = p;
    }
  }
  sk[threadIdx.x] = best;
  sp[threadIdx.x] = bp;
  __syncthreads();
  for (int s = kCommitThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const int op = sp[threadIdx.x + s];
      const double ov = sk[threadIdx.x + s];
      const int mp = sp[threadIdx.x];
      if (op >= 0 && (mp < 0 || ov < sk[threadIdx.x] || (ov == sk[threadIdx.x] && op < mp))) {
        sk[threadIdx.x] = ov;
        sp[threadIdx.x] = op;
      }
    }
    __syncthreads();
  }
  const int pc = sp[0];
  const int m = act_cur[pc];
  if (round_second) {
    // Near-tie guard: the runner-up's k (exact for fully evaluated rows; for rows a pruned
    // round left at +inf, their partial k lb[p] — a lower bound above k* (1 + 1e-9)).
    double v2 = INFINITY;
    for (int p = threadIdx.x; p < u; p += kCommitThreads) {
      if (p == pc) continue;
      double v = k[p];
      if (lb && isinf(v)) v = lb[p];
      v2 = fmin(v2, v);
    }
    s2[threadIdx.x] = v2;
    __syncthreads();
    for (int s = kCommitThreads / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) s2[threadIdx.x] = fmin(s2[threadIdx.x], s2[threadIdx.x + s]);
      __syncthreads();
    }
    if (threadIdx.x == 0) round_second[round] = s2[0];
  }
  if (threadIdx.x == 0) {
    rs->chosen_pos = pc;
    rs->chosen_col = m;
    if (round_k) round_k[round] = sk[0];
    if (order) {
      order[round] = col_var[m];
      if (u == 2) order[round + 1] = col_var[act_cur[1 - pc]];  // ordering.cpp:242
    }
  }
  if (scores)
    for (int p = threadIdx.x; p < u; p += kCommitThreads) scores[col_var[act_cur[p]]] = -k[p];
  if (act_nxt)
    for (int p = threadIdx.x; p < u - 1; p += kCommitThreads) act_nxt[p] = act_cur[p < pc ? p : p + 1];
}

// C_rs <- C_rs - (C_rm C_sm) / C_mm for the remaining r, s (bit-symmetric: the product
// commutes). This is the Gram of the residualised columns (regress_out, ordering.cpp:178-211).
__global__ void update_gram_kernel(const double* C, double* Cn, int64_t ldc, const int* act_nxt, int ur,
                                   const RoundState* rs, const unsigned long long* err) {
  if (*err != kNoError) return;
  const int a = blockIdx.y * blockDim.y + threadIdx.y;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= ur || b >= ur) return;
  const int m = rs->chosen_col;
  const int r = act_nxt[a], s = act_nxt[b];
  // C_sm read from row m (C is bit-symmetric): contiguous over s, where column m would be a
  // strided gather; the product commutes, so C stays bit-symmetric. Cn may be C (in place)
  // or the other buffer of a ping-pong pair (resid_ent then recomputes C_rr itself,
  // gram_update_entry, with these exact operations).
  Cn[static_cast<int64_t>(r) * ldc + s] =
      gram_update_entry(C[static_cast<int64_t>(r) * ldc + s], C[static_cast<int64_t>(r) * ldc + m],
                        C[static_cast<int64_t>(m) * ldc + s], C[static_cast<int64_t>(m) * ldc + m]);
}

// regress_out (ordering.cpp:178-211 -> kernels.cpp:106-121) with the reference's sums.
__global__ void regress_out_kernel(const double* X, int64_t ldx, int64_t n, int exog,
                                   const int* remaining, double* out, int64_t ldo, int* zero_var) {
  __shared__ double buf[kSeqChunk];
  const int lane = threadIdx.x;
  const double* xm = X + static_cast<int64_t>(exog) * ldx;
  const double* xr = X + static_cast<int64_t>(remaining[blockIdx.x]) * ldx;
  const double dn = static_cast<double>(n);
  const double mm = warp_seq_sum(xm, n, buf, [](double v) { return v; }) / dn;
  const double var_m = warp_seq_sum(xm, n, buf, [mm](double v) {
                         const double dv = v - mm;
                         return __dmul_rn(dv, dv);
                       }) / dn;
  if (var_m == 0.0) {
    if (lane == 0) *zero_var = 1;
    return;
  }
  const double mr = warp_seq_sum(xr, n, buf, [](double v) { return v; }) / dn;
  // covariance_pop_given_means: s += (x - mx) * (y - my), left to right
  double s = 0.0;
  for (int64_t t0 = 0; t0 < n; t0 += kSeqChunk / 2) {
    const int len = static_cast<int>(lmin(kSeqChunk / 2, n - t0));
    __syncwarp();
    for (int i = lane; i < len; i += 32) {
      buf[2 * i] = xr[t0 + i];
      buf[2 * i + 1] = xm[t0 + i];
    }
    __syncwarp();
    if (lane == 0)
      for (int i = 0; i < len; ++i) s = __dadd_rn(s, __dmul_rn(buf[2 * i] - mr, buf[2 * i + 1] - mm));
  }
  s = __shfl_sync(0xffffffffu, s, 0);
  const double slope = (s / dn) / var_m;
  double* o = out + static_cast<int64_t>(blockIdx.x) * ldo;
  for (int64_t t = lane; t < n; t += 32) o[t] = __dsub_rn(xr[t], __dmul_rn(slope, xm[t]));
}

}  // namespace

void launch_standardize(const double* X, int64_t ldx, int64_t n, const int* col_map, int ncol,
                        double* W, int64_t ldw, int* stat, double* msd, int check_finite,
                        cudaStream_t s) {
  standardize_kernel<<<(ncol + kStdWarps - 1) / kStdWarps, 32 * kStdWarps, 0, s>>>(
      X, ldx, n, col_map, ncol, W, ldw, stat, msd, check_finite);
}

void launch_gram(const double* W, int64_t ldw, int64_t n, int ncol, double* C, int64_t ldc,
                 double* scratch, cudaStream_t s) {
  const GramPlan g = gram_plan(ncol, n);
  gram_kernel<<<dim3(g.ntiles, g.nchunk), 256, 0, s>>>(W, ldw, n, ncol, C, ldc, g.ntb, g.chunk, scratch);
  if (g.nchunk > 1) gram_reduce_kernel<<<g.ntiles, 256, 0, s>>>(scratch, g.ntiles, g.nchunk, g.ntb, n, ncol, C, ldc);
}

void launch_kreduce(const double* epack, const double* H, int u, int nb, double* k,
                    unsigned long long* err, const unsigned long long* errs, int world,
                    const int* act, double* KN, int d, cudaStream_t s) {
  kreduce_kernel<<<(u + 7) / 8, 256, 0, s>>>(epack, H, u, nb, k, err, errs, world, act, KN, d);
}

void launch_commit(const double* k, const int* act_cur, int* act_nxt, int u, const int* col_var,
                   int* order, int round, double* scores, RoundState* rs,
                   const unsigned long long* err, cudaStream_t s, double* round_k, const double* lb, double* round_second) {
  commit_kernel<<<1, kCommitThreads, 0, s>>>(k, act_cur, act_nxt, u, col_var, order, round, scores,
                                             rs, err, round_k, lb, round_second);
}

void launch_update_gram(const double* C, double* Cn, int64_t ldc, const int* act_nxt, int ur, const RoundState* rs,
                        const unsigned long long* err, cudaStream_t s) {
  const dim3 blk(32, 8);
  const dim3 grd((ur + 31) / 32, (ur + 7) / 8);
  update_gram_kernel<<<grd, blk, 0, s>>>(C, Cn, ldc, act_nxt, ur, rs, err);
}


void launch_regress_out(const double* X, int64_t ldx, int64_t n, int exog, const int* remaining,
                        int r, double* out, int64_t ldo, int* zero_var_flag, cudaStream_t s) {
  regress_out_kernel<<<r, 32, 0, s>>>(X, ldx, n, exog, remaining, out, ldo, zero_var_flag);
}

}  // namespace plg
