// ede_probe.cu — ceiling of the EDE element math alone (no pair data staging), to separate
// the pair kernel's pipeline effects from the math's own FP64-pipe efficiency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2403_03772_b200/csrc ede_probe.cu
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "plg_math.cuh"

using namespace plg;

template <int CH>
__global__ void __launch_bounds__(256) ede_kernel(const double* g_exp, const double2* g_log, int iters,
                                                  double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  load_tables(smem, g_exp, g_log);
  __syncthreads();
  const TabPtr tp = table_ptrs(smem, threadIdx.x & 31);
  double u[CH];
  EdeAcc acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) u[c] = (0.001 * (threadIdx.x + 37 * c) - 1.3) * kUScale;
  const double step = 1.0000001;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      ede_accumulate<false>(u[c], acc[c], tp);
      u[c] = -u[c] * step;  // cheap dependent update, keeps |u| ~ O(1)
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc_lc(acc[c]) + acc_pdf(acc[c]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
void run(const double* de, const double2* dl, double* out, int blocks_per_sm, int sms) {
  cudaFuncSetAttribute(ede_kernel<CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTableBytes);
  const int iters = 4096 / CH * 8;
  const int blocks = sms * blocks_per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  ede_kernel<CH><<<blocks, 256, kTableBytes>>>(de, dl, iters, out);
  cudaEventRecord(a);
  ede_kernel<CH><<<blocks, 256, kTableBytes>>>(de, dl, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double ede = double(blocks) * 256 * iters * CH;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("chains %d  ctas/SM %d (warps/SM %d): %.3e EDE/s = %.1f FP64 instr/clk/SM at 31 instr/EDE\n", CH,
         blocks_per_sm, blocks_per_sm * 8, ede / (ms * 1e-3), ede / (ms * 1e-3) * 31 / sms / (clk * 1e3));
}

int main() {
  std::vector<double> e(kExpN);
  std::vector<double2> l(kLogMasterN);
  for (int j = 0; j < kExpN; ++j) {  // pre-compensated rows (plg_math.cuh exp2_k)
    double v = (double)exp2l((long double)j / kExpN);
    unsigned long long b;
    memcpy(&b, &v, 8);
    b -= (unsigned long long)j << 45;
    memcpy(&e[j], &b, 8);
  }
  for (int j = 0; j < kLogMasterN; ++j) {
    const double c = (j == kLogMasterN - 1) ? 0.5 : (double)(1.0L / (1.0L + ((long double)j + 0.5L) / 128));
    l[j] = make_double2(c, (double)(-logl((long double)c) - logl(2.0L)));
  }
  double* de;
  double2* dl;
  double* out;
  cudaMalloc(&de, e.size() * 8);
  cudaMalloc(&dl, l.size() * 16);
  cudaMalloc(&out, 148 * 8 * 256 * 8);
  cudaMemcpy(de, e.data(), e.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dl, l.data(), l.size() * 16, cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int occ : {1, 2, 3, 4}) {
    run<2>(de, dl, out, occ, sms);
    run<4>(de, dl, out, occ, sms);
    run<8>(de, dl, out, occ, sms);
  }
  return 0;
}
