// Per-kernel cost inside a CUDA graph on this GPU: N back-to-back tiny kernels.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty() {}
__global__ void k_touch(double* p, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 1.0000001 + 1.0;
}
int main() {
  cudaStream_t s; cudaStreamCreate(&s);
  double* d; cudaMalloc(&d, sizeof(double) * (1 << 22)); cudaMemset(d, 0, sizeof(double) * (1 << 22));
  for (int variant = 0; variant < 4; ++variant) {
    const int N = 200;
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < N; ++i) {
      if (variant == 0) k_empty<<<1, 32, 0, s>>>();
      else if (variant == 1) k_touch<<<1, 256, 0, s>>>(d, 256);
      else if (variant == 2) k_touch<<<148, 512, 0, s>>>(d, 148 * 512);
      else k_touch<<<4096, 512, 0, s>>>(d, 4096 * 512);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("variant %d: %.2f us per kernel node\n", variant, ms * 1e3 / (10.0 * N));
  }
  return 0;
}
