// Screening-arithmetic probe (measurement infrastructure, not the product).
//
// 1. Exhaustive accuracy of the FP32 special-function unit instructions the screening pair
//    kernel uses, over every FP32 input of the ranges it feeds them:
//      ex2.approx.ftz.f32 on [-200, 0]: max relative error where the result is normal, max
//        absolute error elsewhere (the exact value is then < 2^-126);
//      lg2.approx.ftz.f32 on [1, 2]: max absolute error;
//    against FP64 exp2 / log2 (errors ~1e-16, negligible at this scale).
// 2. Throughput of the candidate screening element loops (registers only, no memory) next
//    to the FP64 table-driven element (plg_math.cuh), per SM per clock.
//
//    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o screen_probe screen_probe.cu
//    ./screen_probe   (prints one JSON object)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2f(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void atomic_max_pos(unsigned long long* p, double v) {
  atomicMax(p, static_cast<unsigned long long>(__double_as_longlong(v)));
}

__global__ void acc_ex2_kernel(uint32_t count, unsigned long long* out) {
  double rel = 0.0, abse = 0.0, worst_x = 0.0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    const float x = __uint_as_float(0x80000000u | i);
    const double ref = exp2(static_cast<double>(x));
    const double got = static_cast<double>(ex2f(x));
    const double e = fabs(got - ref);
    if (ref >= 0x1p-126) {
      const double r = e / ref;
      if (r > rel) rel = r, worst_x = x;
    } else if (e > abse) {
      abse = e;
    }
  }
  atomic_max_pos(&out[0], rel);
  atomic_max_pos(&out[1], abse);
  (void)worst_x;
}

__global__ void acc_lg2_kernel(uint32_t lo, uint32_t hi, unsigned long long* out) {
  double abse = 0.0, rel = 0.0;
  for (uint32_t b = lo + blockIdx.x * blockDim.x + threadIdx.x; b <= hi; b += gridDim.x * blockDim.x) {
    const float y = __uint_as_float(b);
    const double ref = log2(static_cast<double>(y));
    const double e = fabs(static_cast<double>(lg2f(y)) - ref);
    if (e > abse) abse = e;
    if (ref > 0.0 && e / ref > rel) rel = e / ref;
    // per 1/16 of [1, 2): max abs error (bins out[8..24))
    const int bin = min(15, static_cast<int>((y - 1.0f) * 16.0f));
    atomic_max_pos(&out[8 + bin], e);
  }
  atomic_max_pos(&out[2], abse);
  atomic_max_pos(&out[3], rel);
}

// ---- throughput: one sample pair = both residual directions of one sample ----
constexpr float kC1 = -2.8853900817779268f;  // -2 log2(e)
constexpr float kC2 = -0.72134752044448170f;  // -log2(e) / 2

struct Acc32 {
  float a = 0.f, l = 0.f, p = 0.f;
};

__device__ __forceinline__ void scr_ede(float u, Acc32& s) {
  const float a = fabsf(u);
  const float e1 = ex2f(a * kC1);
  const float l = lg2f(1.0f + e1);
  const float e2 = ex2f((u * u) * kC2);
  s.a += a;
  s.l += l;
  s.p = fmaf(u, e2, s.p);
}

// variant 0: FP32 accumulators only
// variant 1: FP32 chains of 8 samples, then F2F.F64.F32 + DADD into FP64 sums
template <int kVar>
__global__ void thr_scr_kernel(int iters, float s1, float b1, float s2, float b2, double* out) {
  float x = threadIdx.x * 1e-3f, y = 0.5f - threadIdx.x * 1e-3f;
  Acc32 c1, c2;
  double d1a = 0, d1l = 0, d1p = 0, d2a = 0, d2l = 0, d2p = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float u1 = fmaf(-b1, y, x * s1);
      const float u2 = fmaf(-b2, x, y * s2);
      scr_ede(u1, c1);
      scr_ede(u2, c2);
      x += 0.001f;
      y -= 0.0007f;
    }
    if (kVar == 1) {
      d1a += c1.a, d1l += c1.l, d1p += c1.p, d2a += c2.a, d2l += c2.l, d2p += c2.p;
      c1 = Acc32{}, c2 = Acc32{};
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] =
      d1a + d1l + d1p + d2a + d2l + d2p + c1.a + c1.l + c1.p + c2.a + c2.l + c2.p;
}

// candidate v3: residuals in FP64 (|u| summed in FP64), converted to FP32 for the MUFU part
struct Acc3 {
  double a = 0.0;
  float l = 0.f, p = 0.f, e1 = 0.f, ae1 = 0.f, ey = 0.f, pabs = 0.f, pq = 0.f;
};
__device__ __forceinline__ void v3_elem(double ud, Acc3& s) {
  s.a += fabs(ud);
  const float u = __double2float_rn(ud);
  const float a = fabsf(u);
  const float e1 = ex2f(__fmul_rn(a, kC1));
  const float y = __fadd_rn(1.0f, e1);
  const float ey = __fsub_rn(e1, __fsub_rn(y, 1.0f));
  const float l = lg2f(y);
  const float q = __fmul_rn(u, u);
  const float p = __fmul_rn(u, ex2f(__fmul_rn(q, kC2)));
  s.l = __fadd_rn(s.l, l);
  s.p = __fadd_rn(s.p, p);
  s.e1 = __fadd_rn(s.e1, e1);
  s.ae1 = fmaf(a, e1, s.ae1);
  s.ey = __fadd_rn(s.ey, fabsf(ey));
  const float pa = fabsf(p);
  s.pabs = __fadd_rn(s.pabs, pa);
  s.pq = fmaf(pa, q, s.pq);
}
__global__ void thr_v3_kernel(int iters, double s1, double b1, double s2, double b2, double* out) {
  double x = threadIdx.x * 1e-3, y = 0.5 - threadIdx.x * 1e-3;
  Acc3 c1, c2;
  double l1 = 0, p1 = 0, l2 = 0, p2 = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v3_elem(fma(y, -b1, x * s1), c1);
      v3_elem(fma(x, -b2, y * s2), c2);
      x += 0.001;
      y -= 0.0007;
    }
    l1 += c1.l, p1 += c1.p, l2 += c2.l, p2 += c2.p;
    c1.l = c1.p = c2.l = c2.p = 0.f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = l1 + p1 + l2 + p2 + c1.a + c2.a + c1.e1 + c1.ae1 + c1.ey + c1.pabs +
                                               c1.pq + c2.e1 + c2.ae1 + c2.ey + c2.pabs + c2.pq;
}

// raw MUFU.EX2 rate
__global__ void thr_mufu_kernel(int iters, double* out) {
  float v0 = threadIdx.x * 1e-6f - 1.f, v1 = v0 - 1, v2 = v0 - 2, v3 = v0 - 3, v4 = v0 - 4, v5 = v0 - 5,
        v6 = v0 - 6, v7 = v0 - 7;
  for (int i = 0; i < iters; ++i) {
    v0 = ex2f(v0) - 1.5f; v1 = ex2f(v1) - 1.5f; v2 = ex2f(v2) - 1.5f; v3 = ex2f(v3) - 1.5f;
    v4 = ex2f(v4) - 1.5f; v5 = ex2f(v5) - 1.5f; v6 = ex2f(v6) - 1.5f; v7 = ex2f(v7) - 1.5f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = v0 + v1 + v2 + v3 + v4 + v5 + v6 + v7;
}

// raw F2F.F64.F32 rate
__global__ void thr_f2f_kernel(int iters, double* out) {
  float v0 = threadIdx.x * 1e-6f, v1 = v0 + 1, v2 = v0 + 2, v3 = v0 + 3, v4 = v0 + 4, v5 = v0 + 5, v6 = v0 + 6,
        v7 = v0 + 7;
  double s = 0;
  for (int i = 0; i < iters; ++i) {
    const double d0 = v0, d1 = v1, d2 = v2, d3 = v3, d4 = v4, d5 = v5, d6 = v6, d7 = v7;
    v0 = static_cast<float>(d0 * 0.5) + 1.f;  // keeps the conversions live; F2F.F32.F64 too
    v1 += 1.f; v2 += 1.f; v3 += 1.f; v4 += 1.f; v5 += 1.f; v6 += 1.f; v7 += 1.f;
    s += d1 + d2 + d3 + d4 + d5 + d6 + d7;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + v0;
}

template <typename K>
float time_kernel(K k, int blocks, int threads) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    k(blocks, threads);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0 && ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  unsigned long long* acc = nullptr;
  cudaMalloc(&acc, 24 * sizeof(unsigned long long));
  cudaMemset(acc, 0, 24 * sizeof(unsigned long long));
  const uint32_t n200 = __builtin_bit_cast(uint32_t, 200.0f);  // |x| <= 200
  acc_ex2_kernel<<<sms * 8, 256>>>(n200 + 1, acc);
  acc_lg2_kernel<<<sms * 8, 256>>>(0x3f800000u, 0x40000000u, acc);
  unsigned long long h[24];
  cudaMemcpy(h, acc, sizeof(h), cudaMemcpyDeviceToHost);
  double e[24];
  for (int i = 0; i < 24; ++i) e[i] = __builtin_bit_cast(double, h[i]);

  double* out = nullptr;
  const int blocks = sms * 8, threads = 256;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  const int it = 4096;
  const double ghz = clk_khz * 1e-6;
  auto per_sm_clk = [&](float ms, double ops_per_thread) {
    return ops_per_thread * blocks * threads / (ms * 1e-3 * ghz * 1e9 * sms);
  };
  const float t0 = time_kernel([&](int b, int t) { thr_scr_kernel<0><<<b, t>>>(it, 1.1f, 0.3f, 1.2f, 0.4f, out); }, blocks, threads);
  const float t1 = time_kernel([&](int b, int t) { thr_scr_kernel<1><<<b, t>>>(it, 1.1f, 0.3f, 1.2f, 0.4f, out); }, blocks, threads);
  const float t3 = time_kernel([&](int b, int t) { thr_v3_kernel<<<b, t>>>(it, 1.1, 0.3, 1.2, 0.4, out); }, blocks, threads);
  printf("{\"v3_samplepairs_per_sm_clk\": %.4f}\n", per_sm_clk(t3, 8.0 * it));
  const float tm = time_kernel([&](int b, int t) { thr_mufu_kernel<<<b, t>>>(it, out); }, blocks, threads);
  const float tf = time_kernel([&](int b, int t) { thr_f2f_kernel<<<b, t>>>(it, out); }, blocks, threads);
  const cudaError_t err = cudaDeviceSynchronize();
  printf("{\"lg2_max_rel_1_2\": %.6e, \"lg2_abs_by_sixteenth\": [", e[3]);
  for (int i = 0; i < 16; ++i) printf("%s%.3e", i ? ", " : "", e[8 + i]);
  printf("]}\n");
  printf("{\"sms\": %d, \"clock_ghz_attr\": %.3f, \"ex2_max_rel\": %.6e, \"ex2_max_rel_log2\": %.3f, "
         "\"ex2_subnormal_max_abs\": %.3e, \"lg2_max_abs_1_2\": %.6e, \"lg2_max_abs_log2\": %.3f, "
         "\"scr_fp32acc_samplepairs_per_sm_clk\": %.4f, \"scr_chain8_f64_samplepairs_per_sm_clk\": %.4f, "
         "\"mufu_ex2_per_sm_clk\": %.3f, \"f2f_f64_f32_per_sm_clk\": %.3f, \"err\": \"%s\"}\n",
         sms, ghz, e[0], log2(e[0]), e[1], e[2], log2(e[2]), per_sm_clk(t0, 8.0 * it), per_sm_clk(t1, 8.0 * it),
         per_sm_clk(tm, 8.0 * it), per_sm_clk(tf, 8.0 * it), cudaGetErrorString(err));
  return 0;
}
