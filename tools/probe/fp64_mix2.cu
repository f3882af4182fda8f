// fp64_mix2.cu — calibrate the issue cost of integer / LDS instructions next to a
// full-rate DFMA stream (2 register pairs per DFMA), 8 independent chains per thread,
// 64 warps per SM.
#include <cstdio>

#define CH 8

template <int INT_PER_8, int LDS_PER_8>
__global__ void k_mix(double* out, int iters, double b) {
  __shared__ double tab[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) tab[i] = i * 1e-3;
  __syncthreads();
  double x[CH], r[CH];
  unsigned y[CH];
  for (int c = 0; c < CH; ++c) {
    x[c] = threadIdx.x * 1e-9 + c;
    r[c] = 0.999 + threadIdx.x * 1e-12 * c;
    y[c] = threadIdx.x * 7 + c;
  }
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], r[c], b);
#pragma unroll
    for (int c = 0; c < INT_PER_8; ++c) y[c] = (y[c] ^ static_cast<unsigned>(i)) & y[(c + 1) % CH];
#pragma unroll
    for (int c = 0; c < LDS_PER_8; ++c) acc += tab[(y[c] + i) & 1023];
  }
  double s = acc;
  for (int c = 0; c < CH; ++c) s += x[c] + r[c] + y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int INT_PER_8, int LDS_PER_8>
void run(const char* name, double* out, int sms, int clk) {
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_mix<INT_PER_8, LDS_PER_8><<<blocks, threads>>>(out, iters, 1e-7);
  cudaEventRecord(e0);
  k_mix<INT_PER_8, LDS_PER_8><<<blocks, threads>>>(out, iters, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dfma = 8.0 * iters * double(blocks) * threads;
  printf("%-22s %.1f DFMA/clk/SM\n", name, dfma / (ms * 1e-3) / sms / (clk * 1e3));
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, sms * 8 * 256 * 8);
  run<0, 0>("dfma only", out, sms, clk);
  run<2, 0>("+ 2 LOP3 / 8 DFMA", out, sms, clk);
  run<4, 0>("+ 4 LOP3 / 8 DFMA", out, sms, clk);
  run<8, 0>("+ 8 LOP3 / 8 DFMA", out, sms, clk);
  run<0, 2>("+ 2 LDS / 8 DFMA", out, sms, clk);
  run<4, 2>("+ 4 LOP3 2 LDS / 8", out, sms, clk);
  return 0;
}
