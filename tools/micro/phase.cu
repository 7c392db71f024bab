// Cycles per bottom-kernel style phase: a Jacobi sweep of an m x m level in
// shared memory by `warps` warps (one point per thread per pass) followed by
// the group barrier; isolates the per-phase floor from the interpreter.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2010_00626_b200/csrc/kc_common.cuh"

__global__ void k_phase(int m, int warps, int iters, long long* out, St9 st) {
  extern __shared__ double sm[];
  const int S = m + 2, tid = threadIdx.x, nth = warps * 32;
  for (int i = tid; i < 3 * S * S; i += blockDim.x) sm[i] = (i % 7) * 0.1;
  __syncthreads();
  if (tid >= nth) return;
  double* u = sm + S + 1;
  double* o = sm + S * S + S + 1;
  const double* f = sm + 2 * S * S + S + 1;
  const float inv = 1.0f / m;
  long long t0 = clock64();
  for (int k = 0; k < iters; ++k) {
    for (int it = tid; it < m * m; it += nth) {
      const int y = (int)(((float)it + 0.5f) * inv), x = it - y * m;
      const double* p = u + y * S + x;
      const double au = kc_sum9(st, p[-S - 1], p[-S], p[-S + 1], p[-1], p[0], p[1], p[S - 1], p[S], p[S + 1]);
      o[y * S + x] = kc_jacobi_pt(p[0], f[y * S + x], au, st.c);
    }
    if (warps == 1) __syncwarp();
    else if (warps == 16) __syncthreads();
    else asm volatile("bar.sync 1, %0;" ::"r"(nth) : "memory");
    double* t = u; u = o; o = t;
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = t1 - t0;
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  St9 st{};
  for (int k = 0; k < 9; ++k) st.w[k] = -0.1;
  st.w[4] = 1.0; st.center = 1.0; st.c = 0.8;
  for (int m : {3, 7, 15, 31}) {
    for (int warps : {1, 2, 4, 8, 16}) {
      const int S = m + 2;
      size_t smem = 3 * S * S * sizeof(double);
      k_phase<<<1, 512, smem>>>(m, warps, 100, d, st);
      k_phase<<<1, 512, smem>>>(m, warps, 1000, d, st);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      printf("m=%2d warps=%2d: %6.0f cycles/phase (%s)\n", m, warps, c / 1000.0, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
