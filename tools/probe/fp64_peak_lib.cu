// In-job FP64 roofline probe for bench.py (measurement infrastructure, not the product):
// the DFMA throughput of this GPU at its current clocks, the denominator of the pair
// kernels' FP64-pipe roofline. Exposed as a plain C function loaded with ctypes.
#include <cuda_runtime.h>

namespace {
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
         x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
}  // namespace

// Best of `reps` timed launches (after one warm-up): DFMA TFLOP/s (2 flops per DFMA) and
// the SM count. Returns 0 on success, the CUDA error code otherwise.
extern "C" int fp64_dfma_peak(int device, int reps, double* tflops, int* sms) {
  if (cudaSetDevice(device) != cudaSuccess) return 1;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  const int blocks = nsm * 8, threads = 256, iters = 1 << 16;
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double) * blocks * threads) != cudaSuccess) return 2;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double best = 0.0;
  for (int rep = -1; rep < reps; ++rep) {
    cudaEventRecord(a);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double tf = 2.0 * 8 * static_cast<double>(iters) * blocks * threads / (ms * 1e-3) / 1e12;
    if (rep >= 0 && tf > best) best = tf;
  }
  const cudaError_t e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  *tflops = best;
  *sms = nsm;
  return e == cudaSuccess ? 0 : static_cast<int>(e);
}
