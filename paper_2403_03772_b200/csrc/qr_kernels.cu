// qr_kernels.cu — FP64 blocked Householder QR in echelon form: DirectLiNGAM's weight step
// (reference proj/src/direct_lingam.cpp:46-70) and the VAR
// front-end's least squares (proj/src/var_lingam.cpp:39-44).
//
// The reference solves one least-squares problem per target with Eigen's
// ColPivHouseholderQR on the centred predecessor design, and falls back to the
// minimum-norm CompleteOrthogonalDecomposition solution when qr.rank() < p. Every
// predecessor design is a column prefix of the order-permuted centred matrix A, so ONE
// Householder QR of A gives all of them: column p's first r coordinates c_p (r = rank of
// the prefix) against the leading triangle.
//
// Rank follows ColPivHouseholderQR::rank(): a column whose residual norm after the
// reflectors of the columns before it is at or below thr[k] (the weight step passes
// eps * min(n, k + 1) * max_{j <= k} ||a_j||, the threshold of the first design column k
// enters) is "dependent" and gets no reflector, so the factor is in echelon form
// A_S = Q_r T. For target p with dependent predecessors D the minimum-norm solution is
// b_I = a - G b_D, b_D = (I + G^T G)^-1 G^T a, with a = T_I^-1 c_p and g_k = T_I^-1 c_k
// (qr_mincorr_kernel): exactly the COD solution of direct_lingam.cpp:62.
//
// Blocking (32-column panels, compact WY):
//   qr_panel_kernel   one thread-block cluster (8 or 16 CTAs, rows split between them)
//                     factors the panel column by column; the per-column norm and dot
//                     products are reduced across the cluster through distributed shared
//                     memory in a fixed order, so every CTA holds identical scalars and the
//                     result is deterministic; it then builds T (I - V T V^T) of the panel.
//   qr_ypart/qr_z/qr_update   trailing matrix A2 <- (I - V T^T V^T) A2 as Y = V^T A2 (row
//                     chunks reduced in ascending order), Z = T^T Y, A2 -= V Z.
//   qr_solve_kernel   a_k = T_I^-1 c_k for every column (warp per column, column-oriented
//                     back substitution in shared memory), scattered into B.
// The number of reflectors is data dependent; it lives on the device (qstate, pinfo), so
// the host enqueues a fixed sequence of launches without synchronising.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "plg_kernels.h"

namespace cg = cooperative_groups;

namespace plg {

namespace {

constexpr int kNB = kQrNB;  // panel width
constexpr int kPT = 256;    // panel kernel threads
constexpr int kPW = kPT / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum in a fixed order (warp trees, then warp 0 over the warp partials).
__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  const int nw = (blockDim.x + 31) >> 5;
  if (threadIdx.x < 32) {
    t = l < nw ? red[l] : 0.0;
    t = warp_sum(t);
  }
  __syncthreads();
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

// A[:, k] = X[:, order[k]] - mean, cn[k] = ||A[:, k]||. order == nullptr: identity.
__global__ void __launch_bounds__(256) qr_center_kernel(const double* X, int64_t ldx, int64_t n, const int* order,
                                                        int center, double* A, int64_t lda, double* cn) {
  __shared__ double red[32];
  const int k = blockIdx.x;
  const double* x = X + static_cast<int64_t>(order ? order[k] : k) * ldx;
  double* a = A + static_cast<int64_t>(k) * lda;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  const double mean = center ? block_sum(s, red) / static_cast<double>(n) : 0.0;
  double q = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = x[i] - mean;
    a[i] = v;
    q += v * v;
  }
  q = block_sum(q, red);
  if (threadIdx.x == 0) cn[k] = sqrt(q);
}

// Weight-step thresholds: thr[k] = eps * min(n, k + 1) * max_{j <= k} cn[j]; qstate = {0, 0}.
__global__ void qr_thr_prefix_kernel(const double* cn, int64_t n, int d, double* thr, int* qstate) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double mx = 0.0;
  for (int k = 0; k < d; ++k) {
    mx = fmax(mx, cn[k]);
    const double dim = static_cast<double>(static_cast<int64_t>(k + 1) < n ? k + 1 : n);
    thr[k] = 2.220446049250313e-16 * dim * mx;
  }
  qstate[0] = 0;
  qstate[1] = 0;
}

// VAR thresholds: one design of ncol columns (rank test of the whole Z, var_lingam.cpp:40),
// response columns never get a reflector.
__global__ void qr_thr_design_kernel(const double* cn, int64_t n, int ncol, int ntot, double* thr, int* qstate) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double mx = 0.0;
  for (int k = 0; k < ncol; ++k) mx = fmax(mx, cn[k]);
  const double dim = static_cast<double>(static_cast<int64_t>(ncol) < n ? ncol : n);
  for (int k = 0; k < ntot; ++k) thr[k] = k < ncol ? 2.220446049250313e-16 * dim * mx : INFINITY;
  qstate[0] = 0;
  qstate[1] = 0;
}

// One 32-column panel [k0, k0 + nb) on rows [r, n), r = qstate[0].
__global__ void __launch_bounds__(kPT) qr_panel_kernel(double* A, int64_t lda, int64_t n, int ncol, int k0,
                                                       const double* thr, int* qstate, int* rbefore, int* rowcol,
                                                       double* tau, int* dep, int* pinfo, double* Tout) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = static_cast<int>(cl.block_rank());
  const int ncl = static_cast<int>(cl.num_blocks());
  const int nb = min(kNB, ncol - k0);
  const int64_t S = (n + ncl - 1) / ncl;
  const int64_t lo = static_cast<int64_t>(rank) * S;
  const int64_t hi = lo + S < n ? lo + S : n;
  __shared__ double part[2][2 * kNB];
  __shared__ double tot[2 * kNB];
  __shared__ double sl[kNB];
  __shared__ double vpart[kNB * (kNB - 1) / 2];
  __shared__ int pcol[kNB];
  __shared__ double ptau[kNB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int r = qstate[0];
  const int r0 = r;
  int m = 0;
  for (int j = 0; j < nb; ++j) {
    const int k = k0 + j;
    double* ak = A + static_cast<int64_t>(k) * lda;
    const int nit = nb - j;  // item 0: column k (norm); item q: column k + q (dot with column k)
    const int par = j & 1;
    const int64_t tlo = lo > static_cast<int64_t>(r) + 1 ? lo : static_cast<int64_t>(r) + 1;
    const bool own_r = r >= lo && r < hi;
    for (int it = warp; it < nit; it += kPW) {
      const double* al = ak + static_cast<int64_t>(it) * lda;
      double s = 0.0;
      for (int64_t i = tlo + lane; i < hi; i += 32) s += ak[i] * al[i];
      s = warp_sum(s);
      if (lane == 0) {
        part[par][2 * it] = s;
        part[par][2 * it + 1] = own_r ? al[r] : 0.0;
      }
    }
    cl.sync();
    if (threadIdx.x < 2 * nit) {
      double t = 0.0;
      for (int q = 0; q < ncl; ++q) t += cl.map_shared_rank(&part[par][0], q)[threadIdx.x];
      tot[threadIdx.x] = t;
    }
    __syncthreads();
    const double tail = tot[0], c0 = tot[1];
    const double nu = sqrt(c0 * c0 + tail);
    const bool indep = static_cast<int64_t>(r) < n && nu > thr[k];
    if (indep) {
      double beta = c0 >= 0.0 ? -nu : nu, tk = 0.0, denom = 1.0;
      if (tail == 0.0) {
        beta = c0;
      } else {
        denom = c0 - beta;
        tk = (beta - c0) / beta;
      }
      if (threadIdx.x > 0 && threadIdx.x < nit) sl[threadIdx.x] = tk * (tot[2 * threadIdx.x + 1] + tot[2 * threadIdx.x] / denom);
      __syncthreads();
      for (int64_t i = tlo + threadIdx.x; i < hi; i += kPT) {
        const double v = ak[i] / denom;
        ak[i] = v;
        for (int q = 1; q < nit; ++q) ak[static_cast<int64_t>(q) * lda + i] -= sl[q] * v;
      }
      if (own_r && threadIdx.x == 0) {
        ak[r] = beta;
        for (int q = 1; q < nit; ++q) ak[static_cast<int64_t>(q) * lda + r] -= sl[q];
      }
      if (threadIdx.x == 0) {
        pcol[m] = k;
        ptau[m] = tk;
        if (rank == 0) {
          rbefore[k] = r;
          rowcol[r] = k;
          tau[k] = tk;
          dep[k] = 0;
        }
      }
      ++m;
      ++r;
    } else if (threadIdx.x == 0 && rank == 0) {
      rbefore[k] = r;
      tau[k] = 0.0;
      dep[k] = 1;
      ++qstate[1];
    }
    __syncthreads();
  }
  // V^T V (strict upper part) for T: v_t = e_{r0+t} + A[r0+t+1:, pcol[t]]
  const int np = m * (m - 1) / 2;
  for (int pq = warp; pq < np; pq += kPW) {
    int t = 1, base = 0;
    while (base + t <= pq) {
      base += t;
      ++t;
    }
    const int s_ = pq - base;  // s_ < t
    const double* vs = A + static_cast<int64_t>(pcol[s_]) * lda;
    const double* vt = A + static_cast<int64_t>(pcol[t]) * lda;
    const int64_t rt = r0 + t;
    double acc = 0.0;
    const int64_t b = lo > rt + 1 ? lo : rt + 1;
    for (int64_t i = b + lane; i < hi; i += 32) acc += vs[i] * vt[i];
    acc = warp_sum(acc);
    if (lane == 0) vpart[pq] = acc + ((rt >= lo && rt < hi) ? vs[rt] : 0.0);
  }
  cl.sync();
  if (rank == 0) {
    __shared__ double vtv[kNB * (kNB - 1) / 2];
    __shared__ double T[kNB][kNB];
    for (int pq = threadIdx.x; pq < np; pq += kPT) {
      double t = 0.0;
      for (int q = 0; q < ncl; ++q) t += cl.map_shared_rank(&vpart[0], q)[pq];
      vtv[pq] = t;
    }
    for (int e = threadIdx.x; e < kNB * kNB; e += kPT) T[e / kNB][e % kNB] = 0.0;
    __syncthreads();
    if (threadIdx.x == 0) {
      // forward compact WY: T[t][t] = tau_t, T[0:t, t] = -tau_t T[0:t, 0:t] (V^T v_t)[0:t]
      for (int t = 0; t < m; ++t) {
        T[t][t] = ptau[t];
        const int base = t * (t - 1) / 2;
        for (int i = 0; i < t; ++i) {
          double s = 0.0;
          for (int q = i; q < t; ++q) s += T[i][q] * vtv[base + q];
          T[i][t] = -ptau[t] * s;
        }
      }
      pinfo[0] = r0;
      pinfo[1] = m;
      qstate[0] = r;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kNB * kNB; e += kPT) Tout[e] = T[e % kNB][e / kNB];  // column-major
  }
  cl.sync();
}

// v_t[i] of panel reflector t (rows relative to the matrix): 0 above r0 + t, 1 at r0 + t.
__device__ __forceinline__ double vref(const double* A, int64_t lda, const int* rowcol, int r0, int t, int64_t i) {
  const int64_t rt = r0 + t;
  if (i < rt) return 0.0;
  if (i == rt) return 1.0;
  return A[static_cast<int64_t>(rowcol[rt]) * lda + i];
}

constexpr int kYC = 32;   // trailing columns per CTA
constexpr int kYR = 32;   // rows per shared-memory stage

// Ypart[s][t][c] = sum over rows of chunk s (>= r0) of v_t[i] A[i, c0 + c]
__global__ void __launch_bounds__(256) qr_ypart_kernel(const double* A, int64_t lda, int64_t n, int c_begin,
                                                       int ntrail, const int* rowcol, const int* pinfo,
                                                       int64_t chunk, double* Yp) {
  __shared__ double Vs[kYR][kNB + 1];
  __shared__ double As[kYR][kYC + 1];
  const int r0 = pinfo[0], m = pinfo[1];
  const int cb = blockIdx.x * kYC;
  const int s = blockIdx.y;
  const int64_t rs0 = static_cast<int64_t>(s) * chunk;
  const int64_t rbeg = rs0 > r0 ? rs0 : r0;
  const int64_t rend = rs0 + chunk < n ? rs0 + chunk : n;
  const int tid = threadIdx.x;
  const int t2 = (tid >> 4) * 2, c2 = (tid & 15) * 2;  // outputs (t2, t2+1) x (c2, c2+1)
  double acc00 = 0.0, acc01 = 0.0, acc10 = 0.0, acc11 = 0.0;
  for (int64_t i0 = rbeg; i0 < rend; i0 += kYR) {
    __syncthreads();
    for (int e = tid; e < kYR * kNB; e += 256) {
      const int ii = e % kYR, t = e / kYR;
      const int64_t i = i0 + ii;
      Vs[ii][t] = (i < rend && t < m) ? vref(A, lda, rowcol, r0, t, i) : 0.0;
    }
    for (int e = tid; e < kYR * kYC; e += 256) {
      const int ii = e % kYR, c = e / kYR;
      const int64_t i = i0 + ii;
      As[ii][c] = (i < rend && cb + c < ntrail) ? A[static_cast<int64_t>(c_begin + cb + c) * lda + i] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int ii = 0; ii < kYR; ++ii) {
      const double v0 = Vs[ii][t2], v1 = Vs[ii][t2 + 1];
      const double a0 = As[ii][c2], a1 = As[ii][c2 + 1];
      acc00 = fma(v0, a0, acc00);
      acc01 = fma(v0, a1, acc01);
      acc10 = fma(v1, a0, acc10);
      acc11 = fma(v1, a1, acc11);
    }
  }
  double* y = Yp + static_cast<int64_t>(s) * kNB * ntrail;
  const int c = cb + c2;
  if (c < ntrail) {
    y[static_cast<int64_t>(t2) * ntrail + c] = acc00;
    y[static_cast<int64_t>(t2 + 1) * ntrail + c] = acc10;
  }
  if (c + 1 < ntrail) {
    y[static_cast<int64_t>(t2) * ntrail + c + 1] = acc01;
    y[static_cast<int64_t>(t2 + 1) * ntrail + c + 1] = acc11;
  }
}

// Z[t][c] = sum_u T[u][t] * (sum_s Ypart[s][u][c])  (Z = T^T V^T A2)
__global__ void __launch_bounds__(128) qr_z_kernel(const double* Yp, int nsplit, int ntrail, const double* T,
                                                   const int* pinfo, double* Z) {
  __shared__ double Ts[kNB * kNB];
  for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) Ts[e] = T[e];
  __syncthreads();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ntrail) return;
  const int m = pinfo[1];
  double y[kNB];
#pragma unroll
  for (int t = 0; t < kNB; ++t) y[t] = 0.0;
  for (int s = 0; s < nsplit; ++s) {
    const double* p = Yp + static_cast<int64_t>(s) * kNB * ntrail + c;
#pragma unroll
    for (int t = 0; t < kNB; ++t)
      if (t < m) y[t] += p[static_cast<int64_t>(t) * ntrail];
  }
#pragma unroll
  for (int t = 0; t < kNB; ++t) {
    double z = 0.0;
#pragma unroll
    for (int u = 0; u <= t; ++u) z = fma(Ts[t * kNB + u], y[u], z);  // T column-major: T[u][t] at t*kNB+u
    if (t < m) Z[static_cast<int64_t>(t) * ntrail + c] = z;
  }
}

constexpr int kUR = 64;  // rows per update CTA
// A2[i, c] -= sum_t v_t[i] Z[t][c] for rows i >= r0
__global__ void __launch_bounds__(256) qr_update_kernel(double* A, int64_t lda, int64_t n, int c_begin, int ntrail,
                                                        const int* rowcol, const int* pinfo, const double* Z) {
  __shared__ double Vs[kUR][kNB + 1];
  __shared__ double Zs[kNB][kYC + 1];
  const int r0 = pinfo[0], m = pinfo[1];
  if (m == 0) return;
  const int cb = blockIdx.x * kYC;
  const int64_t i0 = static_cast<int64_t>(blockIdx.y) * kUR;
  if (i0 + kUR <= r0) return;
  const int tid = threadIdx.x;
  for (int e = tid; e < kUR * kNB; e += 256) {
    const int ii = e % kUR, t = e / kUR;
    const int64_t i = i0 + ii;
    Vs[ii][t] = (i < n && t < m) ? vref(A, lda, rowcol, r0, t, i) : 0.0;
  }
  for (int e = tid; e < kNB * kYC; e += 256) {
    const int c = e % kYC, t = e / kYC;
    Zs[t][c] = (t < m && cb + c < ntrail) ? Z[static_cast<int64_t>(t) * ntrail + cb + c] : 0.0;
  }
  __syncthreads();
  // thread: row ii = tid % 64, columns (tid / 64) * 8 .. + 8
  const int ii = tid % kUR, cq = (tid / kUR) * 8;
  const int64_t i = i0 + ii;
  if (i < r0 || i >= n) return;
  double acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.0;
  for (int t = 0; t < m; ++t) {
    const double v = Vs[ii][t];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = fma(v, Zs[t][cq + q], acc[q]);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c = cb + cq + q;
    if (c < ntrail) A[static_cast<int64_t>(c_begin + c) * lda + i] -= acc[q];
  }
}

// a_k = T_I^-1 c_k for column k (rows 0..rbefore[k]); warp per column, shared memory.
// With B != nullptr, coefficient t of column k goes to B[order[k] + ldb * order[rowcol[t]]]
// (weights), or with order == nullptr to B[rowcol[t] + ldb * (k - k_first)] (VAR).
__global__ void qr_solve_kernel(const double* A, int64_t lda, int ncol, int k_first, const int* rbefore,
                                const int* rowcol, double* coef, int64_t ldcoef, const int* order, double* B,
                                int64_t ldb) {
  extern __shared__ double sc[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = k_first + blockIdx.x * (blockDim.x >> 5) + w;
  if (k >= ncol) return;
  double* a = sc + static_cast<int64_t>(w) * ldcoef;
  const int r = rbefore[k];
  const double* ck = A + static_cast<int64_t>(k) * lda;
  for (int i = lane; i < r; i += 32) a[i] = ck[i];
  __syncwarp();
  for (int t = r - 1; t >= 0; --t) {
    const double* col = A + static_cast<int64_t>(rowcol[t]) * lda;
    const double at = a[t] / col[t];
    for (int i = lane; i < t; i += 32) a[i] -= at * col[i];
    __syncwarp();
    if (lane == 0) a[t] = at;
    __syncwarp();
  }
  double* out = coef + static_cast<int64_t>(k) * ldcoef;
  for (int i = lane; i < r; i += 32) {
    out[i] = a[i];
    if (B && order) B[order[k] + ldb * order[rowcol[i]]] = a[i];           // weights: B[target, pred]
    else if (B) B[rowcol[i] + ldb * static_cast<int64_t>(k - k_first)] = a[i];  // VAR: coef[pred, response]
  }
}

// Targets with dependent predecessors: minimum-norm correction (see the header comment).
// deps: ascending dependent columns; tg: the targets (one per CTA); mcount[b]: dependent
// predecessors of tg[b]; N: per-CTA scratch of mmax * mmax doubles.
__global__ void __launch_bounds__(256) qr_mincorr_kernel(const double* coef, int64_t ldcoef, const int* rbefore,
                                                         const int* rowcol, const int* deps, const int* tg,
                                                         const int* mcount, const int* order, double* N, int mmax,
                                                         double* B, int64_t ldb) {
  extern __shared__ double sh[];  // y[mmax]
  const int p = tg[blockIdx.x];
  const int m = mcount[blockIdx.x];
  double* Nb = N + static_cast<int64_t>(blockIdx.x) * mmax * mmax;
  double* y = sh;
  const double* a = coef + static_cast<int64_t>(p) * ldcoef;
  const int rp = rbefore[p];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // N = I + G^T G (lower triangle), y = G^T a
  const int ntri = m * (m + 1) / 2;
  for (int e = w; e < ntri + m; e += nw) {
    if (e < ntri) {
      int i = 0, base = 0;
      while (base + i + 1 <= e) {
        base += i + 1;
        ++i;
      }
      const int j = e - base;  // j <= i
      const double* gi = coef + static_cast<int64_t>(deps[i]) * ldcoef;
      const double* gj = coef + static_cast<int64_t>(deps[j]) * ldcoef;
      const int ri = rbefore[deps[i]], rj = rbefore[deps[j]];
      const int rm = ri < rj ? ri : rj;
      double s = 0.0;
      for (int t = lane; t < rm; t += 32) s += gi[t] * gj[t];
      s = warp_sum(s);
      if (lane == 0) Nb[static_cast<int64_t>(i) * mmax + j] = s + (i == j ? 1.0 : 0.0);
    } else {
      const int i = e - ntri;
      const double* gi = coef + static_cast<int64_t>(deps[i]) * ldcoef;
      const int ri = rbefore[deps[i]];
      double s = 0.0;
      for (int t = lane; t < ri; t += 32) s += gi[t] * a[t];
      s = warp_sum(s);
      if (lane == 0) y[i] = s;
    }
  }
  __syncthreads();
  // Cholesky (right-looking, lower), then the two triangular solves
  for (int j = 0; j < m; ++j) {
    const double l = sqrt(Nb[static_cast<int64_t>(j) * mmax + j]);
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) Nb[static_cast<int64_t>(i) * mmax + j] /= l;
    if (threadIdx.x == 0) Nb[static_cast<int64_t>(j) * mmax + j] = l;
    __syncthreads();
    const int rem = m - j - 1;
    for (int e = threadIdx.x; e < rem * rem; e += blockDim.x) {
      const int i = j + 1 + e / rem, q = j + 1 + e % rem;
      if (q <= i)
        Nb[static_cast<int64_t>(i) * mmax + q] -=
            Nb[static_cast<int64_t>(i) * mmax + j] * Nb[static_cast<int64_t>(q) * mmax + j];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < m; ++i) {
      double t = y[i];
      for (int q = 0; q < i; ++q) t -= Nb[static_cast<int64_t>(i) * mmax + q] * y[q];
      y[i] = t / Nb[static_cast<int64_t>(i) * mmax + i];
    }
    for (int i = m - 1; i >= 0; --i) {
      double t = y[i];
      for (int q = i + 1; q < m; ++q) t -= Nb[static_cast<int64_t>(q) * mmax + i] * y[q];
      y[i] = t / Nb[static_cast<int64_t>(i) * mmax + i];
    }
  }
  __syncthreads();
  const int target = order[p];
  for (int t = threadIdx.x; t < rp; t += blockDim.x) {
    double b = a[t];
    for (int i = 0; i < m; ++i) {
      const int ri = rbefore[deps[i]];
      if (t < ri) b -= coef[static_cast<int64_t>(deps[i]) * ldcoef + t] * y[i];
    }
    B[target + ldb * order[rowcol[t]]] = b;
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) B[target + ldb * order[deps[i]]] = y[i];
}

int g_cluster[64];  // per device: chosen cluster size (0 = not yet probed)

}  // namespace

void launch_qr_center(const double* X, int64_t ldx, int64_t n, const int* order, int ncol, int center, double* A,
                      int64_t lda, double* cn, cudaStream_t s) {
  qr_center_kernel<<<ncol, 256, 0, s>>>(X, ldx, n, order, center, A, lda, cn);
}

void launch_qr_thr_prefix(const double* cn, int64_t n, int d, double* thr, int* qstate, cudaStream_t s) {
  qr_thr_prefix_kernel<<<1, 1, 0, s>>>(cn, n, d, thr, qstate);
}

void launch_qr_thr_design(const double* cn, int64_t n, int ncol, int ntot, double* thr, int* qstate, cudaStream_t s) {
  qr_thr_design_kernel<<<1, 1, 0, s>>>(cn, n, ncol, ntot, thr, qstate);
}

int64_t qr_ysplit(int64_t n, int ntrail, int64_t* chunk) {
  const int ctiles = (ntrail + kYC - 1) / kYC;
  int64_t split = (2 * 148 + ctiles - 1) / ctiles;
  const int64_t cap = (n + 255) / 256;
  if (split > cap) split = cap;
  if (split < 1) split = 1;
  *chunk = ((n + split - 1) / split + kYR - 1) / kYR * kYR;
  return (n + *chunk - 1) / *chunk;
}

cudaError_t launch_qr_factor(double* A, int64_t lda, int64_t n, int ncol, const double* thr, int* qstate,
                             int* rbefore, int* rowcol, double* tau, int* dep, int* pinfo, double* T, double* Yp,
                             double* Z, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  int& cls = g_cluster[dev & 63];
  if (cls == 0) {
    cls = 8;
    if (cudaFuncSetAttribute(qr_panel_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 16;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(16);
      cfg.blockDim = dim3(kPT);
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, qr_panel_kernel, &cfg) == cudaSuccess && nclusters > 0) cls = 16;
    }
    cudaGetLastError();
  }
  for (int k0 = 0; k0 < ncol; k0 += kNB) {
    const int panel = k0 / kNB;
    int* pi = pinfo + 2 * panel;
    double* Tp = T + static_cast<int64_t>(panel) * kNB * kNB;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cls;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cls);
    cfg.blockDim = dim3(kPT);
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, qr_panel_kernel, A, lda, n, ncol, k0, thr, qstate, rbefore, rowcol, tau,
                                       dep, pi, Tp);
    if (e != cudaSuccess) return e;
    const int c_begin = k0 + kNB;
    const int ntrail = ncol - c_begin;
    if (ntrail <= 0) continue;
    int64_t chunk = 0;
    const int64_t split = qr_ysplit(n, ntrail, &chunk);
    const int ctiles = (ntrail + kYC - 1) / kYC;
    qr_ypart_kernel<<<dim3(ctiles, static_cast<unsigned>(split)), 256, 0, s>>>(A, lda, n, c_begin, ntrail, rowcol, pi,
                                                                                chunk, Yp);
    qr_z_kernel<<<(ntrail + 127) / 128, 128, 0, s>>>(Yp, static_cast<int>(split), ntrail, Tp, pi, Z);
    qr_update_kernel<<<dim3(ctiles, static_cast<unsigned>((n + kUR - 1) / kUR)), 256, 0, s>>>(A, lda, n, c_begin,
                                                                                           ntrail, rowcol, pi, Z);
  }
  return cudaGetLastError();
}

int64_t qr_yp_doubles(int64_t n, int ncol) {  // the largest Yp over the panels' trailing widths
  int64_t mx = 0;
  for (int k0 = 0; k0 < ncol; k0 += kNB) {
    const int ntrail = ncol - (k0 + kNB);
    if (ntrail <= 0) break;
    int64_t chunk = 0;
    const int64_t split = qr_ysplit(n, ntrail, &chunk);
    mx = std::max<int64_t>(mx, split * kNB * ntrail);
  }
  return mx;
}

int64_t qr_scratch_doubles(int64_t n, int ncol) {
  return qr_yp_doubles(n, ncol) + static_cast<int64_t>(kNB) * ncol;  // Yp + Z
}

cudaError_t launch_qr_solve(const double* A, int64_t lda, int ncol, int k_first, const int* rbefore, const int* rowcol,
                            double* coef, int64_t ldcoef, const int* order, double* B, int64_t ldb, cudaStream_t s) {
  if (k_first >= ncol) return cudaSuccess;
  const size_t per_warp = static_cast<size_t>(ldcoef) * sizeof(double);
  int warps = static_cast<int>(std::min<size_t>(8, (200 * 1024) / std::max<size_t>(per_warp, 1)));
  if (warps < 1) return cudaErrorInvalidValue;  // more than 25 600 columns: not supported
  const size_t smem = per_warp * warps;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(qr_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const int nk = ncol - k_first;
  qr_solve_kernel<<<(nk + warps - 1) / warps, 32 * warps, smem, s>>>(A, lda, ncol, k_first, rbefore, rowcol, coef,
                                                                     ldcoef, order, B, ldb);
  return cudaGetLastError();
}

cudaError_t launch_qr_mincorr(const double* coef, int64_t ldcoef, const int* rbefore, const int* rowcol,
                              const int* deps, const int* tg, const int* mcount, int ntg, const int* order, double* N,
                              int mmax, double* B, int64_t ldb, cudaStream_t s) {
  if (ntg <= 0) return cudaSuccess;
  const size_t smem = static_cast<size_t>(mmax) * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(qr_mincorr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  qr_mincorr_kernel<<<ntg, 256, smem, s>>>(coef, ldcoef, rbefore, rowcol, deps, tg, mcount, order, N, mmax, B, ldb);
  return cudaGetLastError();
}

}  // namespace plg
