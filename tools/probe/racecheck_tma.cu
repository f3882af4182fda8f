// Does compute-sanitizer racecheck model mbarrier-ordered cp.async.bulk rings? (evidence for
// profiles/r2_sanitizer/README.md). Two versions of the same 2-slot ring (one producer warp
// filling slots with cp.async.bulk, consumer warps reading them):
//   mode 0: full/empty mbarriers (the pair_kernel protocol; CUTLASS PipelineTmaAsync's)
//   mode 1: the same plus a __syncthreads() + fence.proxy.async between reading a slot and
//           refilling it (CTA-barrier ordering racecheck understands)
// Results are checked on the host: a real race would corrupt the sums.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(sa(b)), "r"(parity) : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
               "l"(src), "r"(bytes), "r"(sa(bar)) : "memory");
}

constexpr int kChunk = 256, kSlots = 2, kConsumers = 4;
__global__ void ring(const double* in, int nch, double* out, int mode) {
  __shared__ __align__(128) double buf[kSlots][kChunk];
  __shared__ uint64_t full[kSlots], empty[kSlots];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], kConsumers);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double acc = 0.0;
  for (int c = 0; c < nch; ++c) {
    const int s = c % kSlots;
    if (warp == kConsumers) {  // producer
      if (mode == 0 && c >= kSlots) mbar_wait(&empty[s], ((c / kSlots) - 1) & 1);
      if (lane == 0) {
        mbar_expect_tx(&full[s], kChunk * 8);
        bulk(buf[s], in + static_cast<int64_t>(c) * kChunk, kChunk * 8, &full[s]);
      }
      __syncwarp();
    } else {
      mbar_wait(&full[s], (c / kSlots) & 1);
      for (int i = threadIdx.x; i < kChunk; i += 32 * kConsumers) acc += buf[s][i];
      __syncwarp();
      if (mode == 0 && lane == 0) mbar_arrive(&empty[s]);
    }
    if (mode == 1) {
      __syncthreads();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
  }
  if (warp < kConsumers) atomicAdd(out, acc);
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  const int nch = 64;
  double *in, *out;
  cudaMallocManaged(&in, sizeof(double) * nch * kChunk);
  cudaMallocManaged(&out, sizeof(double));
  double ref = 0.0;
  for (int i = 0; i < nch * kChunk; ++i) in[i] = i % 7, ref += i % 7;
  int bad = 0;
  for (int mode = 0; mode < 2; ++mode) {
    if (only >= 0 && mode != only) continue;
    *out = 0.0;
    ring<<<1, 32 * (kConsumers + 1)>>>(in, nch, out, mode);
    cudaDeviceSynchronize();
    printf("mode %d: sum %.1f (expected %.1f) %s\n", mode, *out, ref, *out == ref ? "ok" : "WRONG");
    bad += *out != ref;
  }
  return bad;
}
