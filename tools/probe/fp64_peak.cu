// FP64 pipe microbenchmark: measures DFMA throughput (the pair kernel's roofline denominator).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void exp_kernel(double* out, int iters) {
  double s = 0, x = -threadIdx.x * 1e-3;
  for (int i = 0; i < iters; ++i) { s += log1p(exp(x)) + exp(-0.5 * x * x); x -= 1e-6; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("name=%s sms=%d clock_khz=%d smem_optin=%zu l2=%d\n", p.name, p.multiProcessorCount, clk, p.sharedMemPerBlockOptin, p.l2CacheSize);
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * 8);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 1 << 16;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a); dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 8 * (double)iters * blocks * threads;
    printf("dfma: %.3f ms  %.2f TFLOP/s  (%.3f DFMA/clk/SM at %.0f MHz nominal)\n", ms, flops / ms / 1e9, flops / 2 / (ms * 1e-3) / p.multiProcessorCount / (clk * 1e3), clk / 1e3);
  }
  int it2 = 1 << 12;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a); exp_kernel<<<blocks, threads>>>(out, it2); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double evals = (double)it2 * blocks * threads;
    printf("libdevice log1p(exp)+exp: %.3f ms  %.3e evals/s\n", ms, evals / ms * 1e3);
  }
  return 0;
}
