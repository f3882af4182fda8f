// fp64_mix.cu — FP64-pipe throughput under different operand/instruction mixes (B200).
// Each kernel runs 8 independent chains per thread, 2048 threads per SM.
#include <cstdio>

#define CHAINS 8

// 1 register pair per DFMA (a, b uniform)
__global__ void k_dfma_uniform(double* out, int iters, double a, double b) {
  double x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  double s = 0;
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 3 distinct register pairs per DFMA
__global__ void k_dfma_3reg(double* out, int iters, double a0, double b0) {
  double x[CHAINS], a[CHAINS], b[CHAINS];
  for (int c = 0; c < CHAINS; ++c) {
    x[c] = threadIdx.x * 1e-9 + c;
    a[c] = a0 + threadIdx.x * 1e-12 * c;
    b[c] = b0 - threadIdx.x * 1e-12 * c;
  }
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a[c], b[c]);
  double s = 0;
  for (int c = 0; c < CHAINS; ++c) s += x[c] + a[c] + b[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 2 distinct register pairs (Horner-like: p = fma(p, r, const))
__global__ void k_dfma_2reg(double* out, int iters, double b) {
  double x[CHAINS], r[CHAINS];
  for (int c = 0; c < CHAINS; ++c) {
    x[c] = threadIdx.x * 1e-9 + c;
    r[c] = 0.999 + threadIdx.x * 1e-12 * c;
  }
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], r[c], b);
  double s = 0;
  for (int c = 0; c < CHAINS; ++c) s += x[c] + r[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// DADD chains (1 reg pair + uniform)
__global__ void k_dadd(double* out, int iters, double b) {
  double x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = x[c] + b;
  double s = 0;
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// DFMA + one integer op on an independent register per DFMA
__global__ void k_dfma_int(double* out, int iters, double a, double b) {
  double x[CHAINS];
  unsigned y[CHAINS];
  for (int c = 0; c < CHAINS; ++c) {
    x[c] = threadIdx.x * 1e-9 + c;
    y[c] = threadIdx.x * 7 + c;
  }
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      x[c] = fma(x[c], a, b);
      y[c] = (y[c] ^ 0x9e3779b9u) + (y[c] >> 3);
    }
  double s = 0;
  for (int c = 0; c < CHAINS; ++c) s += x[c] + y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
void time_it(const char* name, F launch, double fp64_per_thread_iter, int blocks, int threads, int iters, int sms,
             int clk) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = fp64_per_thread_iter * iters * double(blocks) * threads;
  printf("%-14s %.1f FP64 instr/clk/SM\n", name, ops / (ms * 1e-3) / sms / (clk * 1e3));
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, sms * 8 * 256 * 8);
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  time_it("dfma_uniform", [&] { k_dfma_uniform<<<blocks, threads>>>(out, iters, 0.999999, 1e-7); }, CHAINS, blocks,
          threads, iters, sms, clk);
  time_it("dfma_2reg", [&] { k_dfma_2reg<<<blocks, threads>>>(out, iters, 1e-7); }, CHAINS, blocks, threads, iters,
          sms, clk);
  time_it("dfma_3reg", [&] { k_dfma_3reg<<<blocks, threads>>>(out, iters, 0.999999, 1e-7); }, CHAINS, blocks,
          threads, iters, sms, clk);
  time_it("dadd", [&] { k_dadd<<<blocks, threads>>>(out, iters, 1e-7); }, CHAINS, blocks, threads, iters, sms, clk);
  time_it("dfma+int", [&] { k_dfma_int<<<blocks, threads>>>(out, iters, 0.999999, 1e-7); }, CHAINS, blocks, threads,
          iters, sms, clk);
  return 0;
}
