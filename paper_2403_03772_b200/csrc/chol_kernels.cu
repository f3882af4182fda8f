// chol_kernels.cu — FP64 blocked Cholesky and the predecessor regressions of DirectLiNGAM's
// weight step (reference proj/src/direct_lingam.cpp:46-70).
//
// With S = P^T Sigma P the order-permuted covariance and S = L L^T, the least-squares
// coefficients of position p on positions 0..p-1 solve L_p^T beta = l_p (L_p the leading
// p x p block, l_p = L[p, 0:p]) — every target's regression from one factorisation.
//
// Blocked right-looking Cholesky (64-wide panels): the diagonal block is factored by one
// CTA in shared memory, the panel below by a row-parallel triangular solve, the trailing
// matrix by a tiled rank-64 update. A pivot that is not positive relative to its original
// diagonal (<= tol * S_jj) stops the factorisation: the design of every later target is
// rank deficient and the host takes the minimum-norm route for those.
#include <cuda_runtime.h>

#include "plg_kernels.h"

namespace plg {

namespace {

constexpr int kNB = 64;

// S[i][j] = C[order[i]][order[j]] (column-major, lds = n).
__global__ void permute_kernel(const double* C, int64_t ldc, const int* order, int n, double* S) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i < n) S[static_cast<int64_t>(j) * n + i] = C[static_cast<int64_t>(order[j]) * ldc + order[i]];
}

// Factor the kNB x kNB diagonal block at k0 (lower triangle) in shared memory.
__global__ void __launch_bounds__(256) potrf_diag_kernel(double* S, int n, int k0, double tol, int* fail) {
  __shared__ double a[kNB][kNB + 1];
  __shared__ int bad;
  const int nb = min(kNB, n - k0);
  if (threadIdx.x == 0) bad = *fail;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int r = e % nb, c = e / nb;
    a[r][c] = S[static_cast<int64_t>(k0 + c) * n + k0 + r];
  }
  __syncthreads();
  if (bad < n) return;  // an earlier block already failed
  for (int j = 0; j < nb; ++j) {
    if (threadIdx.x == 0) {  // S is a correlation matrix: pivots are partial variances <= 1
      double djj = a[j][j];
      for (int k = 0; k < j; ++k) djj -= a[j][k] * a[j][k];
      if (!(djj > tol) && bad == n) bad = k0 + j;
      a[j][j] = djj > 0.0 ? sqrt(djj) : 0.0;
    }
    __syncthreads();
    if (bad < n) break;
    for (int i = j + 1 + threadIdx.x; i < nb; i += blockDim.x) {
      double s = a[i][j];
      for (int k = 0; k < j; ++k) s -= a[i][k] * a[j][k];
      a[i][j] = s / a[j][j];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && bad < n) *fail = bad;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int r = e % nb, c = e / nb;
    if (r >= c) S[static_cast<int64_t>(k0 + c) * n + k0 + r] = a[r][c];
  }
}

// Panel below the diagonal block: row i of A21 solves x L11^T = a (forward substitution).
__global__ void __launch_bounds__(128) trsm_panel_kernel(double* S, int n, int k0, const int* fail) {
  __shared__ double l[kNB][kNB + 1];
  if (*fail < n) return;
  const int nb = min(kNB, n - k0);
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int r = e % nb, c = e / nb;
    l[r][c] = S[static_cast<int64_t>(k0 + c) * n + k0 + r];
  }
  __syncthreads();
  const int i = k0 + nb + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x[kNB];
#pragma unroll 4
  for (int c = 0; c < nb; ++c) {
    double s = S[static_cast<int64_t>(k0 + c) * n + i];
    for (int k = 0; k < c; ++k) s -= x[k] * l[c][k];
    x[c] = s / l[c][c];
  }
  for (int c = 0; c < nb; ++c) S[static_cast<int64_t>(k0 + c) * n + i] = x[c];
}

// Trailing update S22 -= L21 L21^T on the lower triangle, 64x64 tiles, K = panel width.
__global__ void __launch_bounds__(256) syrk_update_kernel(double* S, int n, int k0, int ntb, const int* fail) {
  constexpr int kKH = kNB / 2;  // K in two halves keeps static shared memory under 48 KB
  __shared__ double As[kNB][kKH + 1];
  __shared__ double Bs[kNB][kKH + 1];
  if (*fail < n) return;
  const int k1 = k0 + kNB;
  int bi, bj;  // bi <= bj: tile rows bj, cols bi of the trailing lower triangle
  tile_decode(blockIdx.x, ntb, bi, bj);
  const int r0 = k1 + bj * kNB, c0 = k1 + bi * kNB;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  for (int kh = 0; kh < kNB; kh += kKH) {
    __syncthreads();
    for (int e = threadIdx.x; e < kNB * kKH; e += blockDim.x) {
      const int r = e % kNB, k = e / kNB;
      As[r][k] = (r0 + r < n) ? S[static_cast<int64_t>(k0 + kh + k) * n + r0 + r] : 0.0;
      Bs[r][k] = (c0 + r < n) ? S[static_cast<int64_t>(k0 + kh + k) * n + c0 + r] : 0.0;
    }
    __syncthreads();
    for (int k = 0; k < kKH; ++k) {
      double av[4], bv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        av[q] = As[ty * 4 + q][k];
        bv[q] = Bs[tx * 4 + q][k];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int s = 0; s < 4; ++s) acc[q][s] = fma(av[q], bv[s], acc[q][s]);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int r = r0 + ty * 4 + q, c = c0 + tx * 4 + s;
      if (r < n && c < n && r >= c) S[static_cast<int64_t>(c) * n + r] -= acc[q][s];
    }
}

// Warp per target position p (1 <= p < limit): beta solves L_p^T beta = l_p by backward
// substitution (lanes split each dot product, fixed-shape reduction), then
// B[order[p] + ldb * order[q]] = beta_q * sd[order[p]] / sd[order[q]].
__global__ void regress_rows_kernel(const double* L, int n, const int* order, const double* msd, int limit,
                                    double* beta, double* B, int64_t ldb) {
  const int p = 1 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= limit) return;
  double* bp = beta + static_cast<int64_t>(p) * n;  // scratch row
  for (int i = p - 1; i >= 0; --i) {
    double s = 0.0;
    const double* Li = L + static_cast<int64_t>(i) * n;  // column i: L[k][i] for k > i
    for (int k = i + 1 + lane; k < p; k += 32) s += Li[k] * bp[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) bp[i] = (L[static_cast<int64_t>(i) * n + p] - s) / Li[i];
    __syncwarp();
  }
  const int t = order[p];
  const double sdt = msd[2 * t + 1];
  for (int q = lane; q < p; q += 32) {
    const int o = order[q];
    B[t + ldb * o] = bp[q] * sdt / msd[2 * o + 1];
  }
}

}  // namespace

void launch_permute(const double* C, int64_t ldc, const int* order, int n, double* S, cudaStream_t s) {
  permute_kernel<<<dim3((n + 255) / 256, n), 256, 0, s>>>(C, ldc, order, n, S);
}

void launch_cholesky(double* S, int n, double tol, int* fail, cudaStream_t s) {
  for (int k0 = 0; k0 < n; k0 += kNB) {
    potrf_diag_kernel<<<1, 256, 0, s>>>(S, n, k0, tol, fail);
    const int rest = n - k0 - kNB;
    if (rest <= 0) break;
    trsm_panel_kernel<<<(rest + 127) / 128, 128, 0, s>>>(S, n, k0, fail);
    const int ntb = (rest + kNB - 1) / kNB;
    syrk_update_kernel<<<ntb * (ntb + 1) / 2, 256, 0, s>>>(S, n, k0, ntb, fail);
  }
}

void launch_regress_rows(const double* L, int n, const int* order, const double* msd, int limit, double* beta,
                         double* B, int64_t ldb, cudaStream_t s) {
  if (limit <= 1) return;
  regress_rows_kernel<<<(limit - 1 + 7) / 8, 256, 0, s>>>(L, n, order, msd, limit, beta, B, ldb);
}

}  // namespace plg
