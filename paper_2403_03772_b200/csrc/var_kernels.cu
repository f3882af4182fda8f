// var_kernels.cu — VarLiNGAM front-end on the device: the least-squares
// VAR(lag) with intercept of reference proj/src/var_lingam.cpp:7-53, whose residuals feed the
// causal order. The reference solves the stacked design Z = [1, x(t-1), ..., x(t-lag)] with
// one column-pivoted Householder QR; here the normal equations of the unit-diagonal scaled
// design are factorised by the engine's blocked FP64 Cholesky (chol_kernels.cu) and solved
// with one step of iterative refinement, and the residuals Y - Z B are formed on the device.
//
//   A = [Z | Y]  (n_rows x (n_cols + d), column-major)     build_var_design_kernel
//   G = A^T A / n_rows                                     gram_kernel (round_kernels.cu)
//   S = D^-1 G_zz D^-1, R = D^-1 G_zy  (D = sqrt diag G_zz) var_scale_kernel
//   S = L L^T; x = S^-1 R, refined once; B = D^-1 x         launch_cholesky + var_solve_kernel
//   E = Y - Z B                                            var_resid_kernel
#include <cuda_runtime.h>

#include <cstdint>

#include "plg_kernels.h"

namespace plg {

namespace {

// A[c * lda + r]: c = 0 intercept, c = 1 + (tau-1) d + j lag tau of variable j, then Y.
__global__ void build_var_design_kernel(const double* ts, int64_t ldt, int64_t n_rows, int d, int lag,
                                        double* A, int64_t lda, int* nonfinite) {
  const int c = blockIdx.y;
  const int n_cols = 1 + lag * d;
  double* out = A + static_cast<int64_t>(c) * lda;
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < lda;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v = 0.0;
    if (r < n_rows) {
      if (c == 0) {
        v = 1.0;
      } else if (c < n_cols) {
        const int tau = 1 + (c - 1) / d, j = (c - 1) % d;
        v = ts[static_cast<int64_t>(j) * ldt + r + lag - tau];
      } else {
        v = ts[static_cast<int64_t>(c - n_cols) * ldt + r + lag];
      }
      if (!isfinite(v)) atomicExch(nonfinite, 1);
    }
    out[r] = v;
  }
}

// S (n_cols x n_cols) and its untouched copy S0, right-hand sides R (n_cols x d), scales D.
__global__ void var_scale_kernel(const double* G, int64_t ldg, int n_cols, int d, double* S, double* S0, double* R,
                                 double* D) {
  const int j = blockIdx.y;  // column of [S | R]
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_cols; i += gridDim.x * blockDim.x) {
    const double di = sqrt(G[static_cast<int64_t>(i) * ldg + i]);
    if (j == 0) D[i] = di;
    if (j < n_cols) {
      const double v = G[static_cast<int64_t>(j) * ldg + i] / (di * sqrt(G[static_cast<int64_t>(j) * ldg + j]));
      S[static_cast<int64_t>(j) * n_cols + i] = v;
      S0[static_cast<int64_t>(j) * n_cols + i] = v;
    } else {
      R[static_cast<int64_t>(j - n_cols) * n_cols + i] = G[static_cast<int64_t>(j) * ldg + i] / di;
    }
  }
}

// One right-hand side per CTA: x = (L L^T)^-1 b by column-oriented substitutions, then one
// refinement step (r = b - S0 x, dx = (L L^T)^-1 r), then B = x / D.
constexpr int kSolveThreads = 256;
__device__ void chol_solve(const double* L, int n, double* v) {  // v <- (L L^T)^-1 v, in smem
  for (int i = 0; i < n; ++i) {  // L y = v
    __syncthreads();
    const double yi = v[i] / L[static_cast<int64_t>(i) * n + i];
    __syncthreads();
    if (threadIdx.x == 0) v[i] = yi;
    for (int k = i + 1 + threadIdx.x; k < n; k += blockDim.x) v[k] -= L[static_cast<int64_t>(i) * n + k] * yi;
  }
  for (int i = n - 1; i >= 0; --i) {  // L^T x = y
    __syncthreads();
    const double xi = v[i] / L[static_cast<int64_t>(i) * n + i];
    __syncthreads();
    if (threadIdx.x == 0) v[i] = xi;
    for (int k = threadIdx.x; k < i; k += blockDim.x) v[k] -= L[static_cast<int64_t>(k) * n + i] * xi;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kSolveThreads) var_solve_kernel(const double* L, const double* S0, const double* R,
                                                                  const double* D, int n_cols, double* B,
                                                                  const int* fail) {
  extern __shared__ double sm[];
  if (*fail < n_cols) return;
  double* x = sm;
  double* r = sm + n_cols;
  const int e = blockIdx.x;
  const double* b = R + static_cast<int64_t>(e) * n_cols;
  for (int i = threadIdx.x; i < n_cols; i += blockDim.x) x[i] = b[i];
  chol_solve(L, n_cols, x);
  for (int i = threadIdx.x; i < n_cols; i += blockDim.x) {  // residual of the normal equations
    double s = b[i];
    for (int k = 0; k < n_cols; ++k) s -= S0[static_cast<int64_t>(k) * n_cols + i] * x[k];
    r[i] = s;
  }
  chol_solve(L, n_cols, r);
  for (int i = threadIdx.x; i < n_cols; i += blockDim.x)
    B[static_cast<int64_t>(e) * n_cols + i] = (x[i] + r[i]) / D[i];
}

// E[e * lde + row] = Y(row, e) - sum_c Z(row, c) B(c, e): 64 x 64 output tiles, 16-deep
// shared-memory panels, 4 x 4 outputs per thread.
constexpr int kRT = 64, kRK = 16;
__global__ void __launch_bounds__(256) var_resid_kernel(const double* A, int64_t lda, int64_t n_rows, int n_cols,
                                                        int d, const double* B, double* E, int64_t lde) {
  __shared__ double Zs[kRK][kRT + 2];
  __shared__ double Bs[kRK][kRT + 2];
  const int r0 = blockIdx.x * kRT, e0 = blockIdx.y * kRT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < n_cols; k0 += kRK) {
    for (int i = threadIdx.x; i < kRK * kRT; i += 256) {
      const int kk = i / kRT, rr = i % kRT;
      const int64_t row = r0 + rr;
      const int c = k0 + kk;
      Zs[kk][rr] = (row < n_rows && c < n_cols) ? A[static_cast<int64_t>(c) * lda + row] : 0.0;
      const int e = e0 + rr;
      Bs[kk][rr] = (e < d && c < n_cols) ? B[static_cast<int64_t>(e) * n_cols + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kRK; ++kk) {
      double zv[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) zv[a] = Zs[kk][tx + 16 * a], bv[a] = Bs[kk][ty + 16 * a];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(zv[a], bv[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t row = r0 + tx + 16 * a;
      const int e = e0 + ty + 16 * b;
      if (row < n_rows && e < d)
        E[static_cast<int64_t>(e) * lde + row] = A[static_cast<int64_t>(n_cols + e) * lda + row] - acc[a][b];
    }
}

}  // namespace

void launch_build_var_design(const double* ts, int64_t ldt, int64_t n_rows, int d, int lag, double* A, int64_t lda,
                             int* nonfinite, cudaStream_t s) {
  const int ncol = 1 + lag * d + d;
  int gx = static_cast<int>((lda + 255) / 256);
  if (gx > 64) gx = 64;
  build_var_design_kernel<<<dim3(gx, ncol), 256, 0, s>>>(ts, ldt, n_rows, d, lag, A, lda, nonfinite);
}

void launch_var_scale(const double* G, int64_t ldg, int n_cols, int d, double* S, double* S0, double* R, double* D,
                      cudaStream_t s) {
  var_scale_kernel<<<dim3((n_cols + 255) / 256, n_cols + d), 256, 0, s>>>(G, ldg, n_cols, d, S, S0, R, D);
}

void launch_var_solve(const double* L, const double* S0, const double* R, const double* D, int n_cols, int d,
                      double* B, const int* fail, cudaStream_t s) {
  const size_t smem = 2 * static_cast<size_t>(n_cols) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(var_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  var_solve_kernel<<<d, kSolveThreads, smem, s>>>(L, S0, R, D, n_cols, B, fail);
}

void launch_var_resid(const double* A, int64_t lda, int64_t n_rows, int n_cols, int d, const double* B, double* E,
                      int64_t lde, cudaStream_t s) {
  var_resid_kernel<<<dim3(static_cast<unsigned>((n_rows + kRT - 1) / kRT), (d + kRT - 1) / kRT), 256, 0, s>>>(
      A, lda, n_rows, n_cols, d, B, E, lde);
}

}  // namespace plg
