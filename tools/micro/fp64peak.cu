// FP64 pipe throughput on this B200: independent DADD / DMUL / DFMA chains,
// full occupancy, CUDA-event timed.  Gives the FP64-issue roofline used for
// the fused stencil kernels (bit-exact => no FMA contraction).
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(256) k_fp(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) x[k] = __dadd_rn(x[k], a);
      else if (OP == 1) x[k] = __dmul_rn(x[k], b);
      else x[k] = __fma_rn(x[k], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, iters = 4096;
  const char* nm[3] = {"DADD", "DMUL", "DFMA"};
  for (int op = 0; op < 3; ++op) {
    auto fn = op == 0 ? k_fp<0> : (op == 1 ? k_fp<1> : k_fp<2>);
    fn<<<blocks, 256>>>(d, iters, 1e-9, 0.999999);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    fn<<<blocks, 256>>>(d, iters, 1e-9, 0.999999);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * 256 * iters * 8;
    printf("%s: %.2f Tinst/s  (%.1f inst/clk/SM at 1965 MHz)  %s\n", nm[op], ops / (ms * 1e-3) / 1e12,
           ops / (ms * 1e-3) / (sms * 1.965e9), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
