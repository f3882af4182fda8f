// var_kernels.cu — VarLiNGAM front-end on the device: the least-squares
// VAR(lag) with intercept of reference proj/src/var_lingam.cpp:7-53, whose residuals feed the
// causal order. The reference solves the stacked design Z = [1, x(t-1), ..., x(t-lag)] with
// one column-pivoted Householder QR; here the same least squares run through the engine's
// FP64 Householder QR (qr_kernels.cu) and the residuals Y - Z B are formed on the device.
//
//   A = [Z | Y]  (n_rows x (n_cols + d), column-major)     build_var_design_kernel
//   QR of Z (response columns receive the reflectors),
//   B = R^-1 (Q^T Y)                                       qr_kernels.cu
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

void launch_var_resid(const double* A, int64_t lda, int64_t n_rows, int n_cols, int d, const double* B, double* E,
                      int64_t lde, cudaStream_t s) {
  var_resid_kernel<<<dim3(static_cast<unsigned>((n_rows + kRT - 1) / kRT), (d + kRT - 1) / kRT), 256, 0, s>>>(
      A, lda, n_rows, n_cols, d, B, E, lde);
}

}  // namespace plg
