// p2p_kernels.cu — completion signalling of the peer-memory exchange (plg_kernels.h,
// PeerTable). Producers store exchanged values into every rank's arena before these run;
// a signal publishes "this rank's stores of exchange i are done" as the sequence number i
// into every rank's flag slot for this rank (release, system scope), and a wait spins on the
// local arena until every rank's slot reached the next expected number (acquire). The
// counters live in device memory, so captured CUDA graphs replay correctly.
#include <cuda_runtime.h>

#include <cstdint>

#include "plg_kernels.h"

namespace plg {

namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void p2p_signal_kernel(const PeerTable pt, const unsigned long long* err, int64_t err_off) {
  if (threadIdx.x != 0) return;
  unsigned long long* f = reinterpret_cast<unsigned long long*>(pt.base[pt.rank] + kArenaFlags);
  const unsigned long long seq = f[0] + 1;
  f[0] = seq;
  if (err_off >= 0) {
    const unsigned long long e = *err;
    for (int r = 0; r < pt.n; ++r)
      *reinterpret_cast<unsigned long long*>(pt.base[r] + err_off + 8 * pt.rank) = e;
  }
  __threadfence_system();
  for (int r = 0; r < pt.n; ++r)
    st_release_sys(reinterpret_cast<unsigned long long*>(pt.base[r] + kArenaFlags) + 2 + pt.rank, seq);
}

__global__ void p2p_wait_kernel(const PeerTable pt) {
  unsigned long long* f = reinterpret_cast<unsigned long long*>(pt.base[pt.rank] + kArenaFlags);
  const unsigned long long target = f[1] + 1;
  if (threadIdx.x < pt.n) {
    const unsigned long long* slot = f + 2 + threadIdx.x;
    while (ld_acquire_sys(slot) < target) __nanosleep(200);
  }
  __syncthreads();
  if (threadIdx.x == 0) f[1] = target;
  __threadfence();
}

}  // namespace

void launch_p2p_signal(const PeerTable& pt, const unsigned long long* err, int64_t err_off, cudaStream_t s) {
  p2p_signal_kernel<<<1, 32, 0, s>>>(pt, err, err_off);
}

void launch_p2p_wait(const PeerTable& pt, cudaStream_t s) { p2p_wait_kernel<<<1, 32, 0, s>>>(pt); }

}  // namespace plg
