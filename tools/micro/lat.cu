// Microbenchmarks for the bottom-kernel design: fp64 dependent-op latency,
// smem load latency, barrier cost, and one small Jacobi phase (m = 7, 15, 31, 63).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2010_00626_b200/csrc/kc_common.cuh"

__global__ void k_chain(double* out, long long* cyc, double a, double b, int n) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __dadd_rn(x, b); x = __dadd_rn(x, b); x = __dadd_rn(x, b); x = __dadd_rn(x, b); }
  long long t1 = clock64();
  double y = a;
  for (int i = 0; i < n; ++i) { y = __dmul_rn(y, b); y = __dmul_rn(y, b); y = __dmul_rn(y, b); y = __dmul_rn(y, b); }
  long long t2 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) { z = fma(z, b, a); z = fma(z, b, a); z = fma(z, b, a); z = fma(z, b, a); }
  long long t3 = clock64();
  if (threadIdx.x == 0) { out[0] = x + y + z; cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}

__global__ void k_bar(long long* cyc, int n, int mode) {
  __shared__ double s[1024];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  double acc = 0;
  int idx = threadIdx.x;
  for (int i = 0; i < n; ++i) {
    if (mode == 0) __syncthreads();
    else if (mode == 1) __syncwarp();
    else { acc += s[idx]; idx = (int)acc & 1023; }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = (long long)acc; }
}

// one CTA, repeated Jacobi phases on an m x m smem grid with `nth` threads, barrier per phase
__global__ void k_phase(long long* cyc, St9 st, int m, int nphase) {
  extern __shared__ double sm[];
  const int S = m + 2;
  for (int i = threadIdx.x; i < 3 * S * S; i += blockDim.x) sm[i] = (i % 7) * 0.1;
  __syncthreads();
  double* a = sm + S + 1;
  double* b = sm + S * S + S + 1;
  const double* f = sm + 2 * S * S + S + 1;
  const float inv = 1.0f / (float)m;
  long long t0 = clock64();
  for (int ph = 0; ph < nphase; ++ph) {
    double* u = (ph & 1) ? b : a;
    double* o = (ph & 1) ? a : b;
    for (int i = threadIdx.x; i < m * m; i += blockDim.x) {
      const int y = (int)(((float)i + 0.5f) * inv), x = i - y * m;
      const int k = y * S + x;
      o[k] = kc_jacobi_pt(u[k], f[k], kc_apply9(u + k, S, st), st.c);
    }
    if (blockDim.x > 32) __syncthreads(); else __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d; long long* c; long long h[4];
  cudaMalloc(&d, 64); cudaMalloc(&c, 64);
  k_chain<<<1, 32>>>(d, c, 1.0, 1e-9, 1000); cudaDeviceSynchronize();
  k_chain<<<1, 32>>>(d, c, 1.0, 1e-9, 1000);
  cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("dependent fp64 latency (cycles): DADD %.2f DMUL %.2f DFMA %.2f\n", h[0] / 4000.0, h[1] / 4000.0, h[2] / 4000.0);
  for (int mode = 0; mode < 3; ++mode) for (int nt : {32, 256, 512, 1024}) {
    k_bar<<<1, nt>>>(c, 1000, mode); cudaDeviceSynchronize();
    k_bar<<<1, nt>>>(c, 1000, mode);
    cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    printf("%s threads=%4d: %.1f cycles/iter\n", mode == 0 ? "__syncthreads" : (mode == 1 ? "__syncwarp  " : "dep LDS chain"), nt, h[0] / 1000.0);
  }
  St9 st;
  for (int k = 0; k < 9; ++k) st.w[k] = -0.1 * (k + 1);
  st.w[4] = 2.0; st.c = 0.4; st.center = 2.0;
  cudaFuncSetAttribute(k_phase, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  for (int m : {3, 7, 15, 31, 63}) for (int nt : {32, 256, 512, 1024}) {
    int S = m + 2;
    size_t sb = 3 * S * S * 8;
    k_phase<<<1, nt, sb>>>(c, st, m, 200); cudaDeviceSynchronize();
    k_phase<<<1, nt, sb>>>(c, st, m, 200);
    cudaError_t e = cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("jacobi phase m=%2d threads=%4d: %.0f cycles/phase %s\n", m, nt, h[0] / 200.0, e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
