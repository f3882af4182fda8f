// Does programmatic dependent launch shorten a chain of small dependent kernels on B200?
// 20 kernels of ~2 us each (592 CTAs x 256 threads reading/writing 1 MB), captured in a
// CUDA graph, with and without PDL (every kernel triggers its dependents at its start and
// waits for its predecessor before touching memory).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void work(double* a, int n, int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = a[i] * 1.0000001 + 1.0;
}

int main() {
  const int n = 1 << 17, chain = 20, reps = 200;
  double* a;
  cudaMalloc(&a, n * sizeof(double));
  cudaMemset(a, 0, n * sizeof(double));
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int k = 0; k < chain; ++k) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(592);
      cfg.blockDim = dim3(256);
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = pdl ? 1 : 0;
      cudaLaunchKernelEx(&cfg, work, a, n, pdl);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphExec_t ge;
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed pdl=%d\n", pdl); return 1; }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("pdl=%d: %.3f us per kernel (%s)\n", pdl, ms * 1e3 / (reps * chain), cudaGetErrorString(cudaGetLastError()));
  }
  // the same chains launched directly into the stream (no graph)
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r)
      for (int k = 0; k < chain; ++k) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(592);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, work, a, n, pdl);
      }
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("stream pdl=%d: %.3f us per kernel\n", pdl, ms * 1e3 / (reps * chain));
  }
  return 0;
}
