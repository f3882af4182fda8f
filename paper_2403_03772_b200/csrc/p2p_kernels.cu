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

__global__ void p2p_signal_kernel(const PeerTable pt, const unsigned long long* err, int64_t err_off) {
  if (threadIdx.x != 0) return;
  if (err_off >= 0) {
    const unsigned long long e = *err;
    for (int r = 0; r < pt.n; ++r)
      *reinterpret_cast<unsigned long long*>(pt.base[r] + err_off + 8 * pt.rank) = e;
  }
  p2p_signal_dev(pt);
}

__global__ void p2p_wait_kernel(const PeerTable pt) {
  if (threadIdx.x == 0) p2p_wait_dev(pt);
  __syncthreads();
}

}  // namespace

void launch_p2p_signal(const PeerTable& pt, const unsigned long long* err, int64_t err_off, cudaStream_t s) {
  p2p_signal_kernel<<<1, 32, 0, s>>>(pt, err, err_off);
}

void launch_p2p_wait(const PeerTable& pt, cudaStream_t s) { p2p_wait_kernel<<<1, 32, 0, s>>>(pt); }

}  // namespace plg
