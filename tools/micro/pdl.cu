// Programmatic dependent launch inside a CUDA graph: per-node cost of a chain
// of one-wave kernels (each block does some dependent work) with and without
// the PDL attribute (secondary waits with griddepcontrol.wait at its start,
// primary triggers its dependents at its start).
#include <cstdio>
#include <cuda_runtime.h>
template <bool PDL>
__global__ void k_work(double* p, int n, int iters) {
  if (PDL) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
  }
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    double v = p[i];
    for (int k = 0; k < iters; ++k) v = v * 1.0000001 + 1e-9;
    p[i] = v;
  }
}
int main() {
  cudaStream_t s; cudaStreamCreate(&s);
  double* d; cudaMalloc(&d, sizeof(double) * (1 << 24)); cudaMemset(d, 0, sizeof(double) * (1 << 24));
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int iters : {0, 200, 2000}) {
    for (int pdl = 0; pdl < 2; ++pdl) {
      const int N = 200, grid = sms * 4, block = 128;
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int i = 0; i < N; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid); cfg.blockDim = dim3(block); cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
        if (pdl) cudaLaunchKernelEx(&cfg, k_work<true>, d, grid * block, iters);
        else cudaLaunchKernelEx(&cfg, k_work<false>, d, grid * block, iters);
      }
      if (cudaStreamEndCapture(s, &g) != cudaSuccess) { printf("capture failed\n"); return 1; }
      if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return 1; }
      cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a, s);
      for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("iters %4d pdl %d: %.2f us per kernel node (%s)\n", iters, pdl, ms * 1e3 / (10.0 * N),
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
