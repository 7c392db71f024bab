// Floor of a CTA-local Jacobi phase on an m x m shared-memory level (FMA
// build arithmetic when compiled with -DKC_FAST=1): `warps` warps, RB rows
// per item (all loads first, RB independent chains), __syncthreads between
// phases.  Compare with a 16-CTA strip phase (~1.9 k cycles at 31^2).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2010_00626_b200/csrc/kc_common.cuh"

template <int RB>
__global__ void k_phase(int m, int iters, long long* out, St9 st) {
  extern __shared__ double sm[];
  const int S = m + 2, tid = threadIdx.x, nth = blockDim.x;
  for (int i = tid; i < 3 * S * S; i += nth) sm[i] = (i % 7) * 0.1;
  __syncthreads();
  double* u = sm + S + 1;
  double* o = sm + S * S + S + 1;
  const double* f = sm + 2 * S * S + S + 1;
  const int nrb = (m + RB - 1) / RB, nitems = nrb * m;
  const float inv = 1.0f / m;
  long long t0 = clock64();
  for (int k = 0; k < iters; ++k) {
    for (int it = tid; it < nitems; it += nth) {
      const int rb = (int)(((float)it + 0.5f) * inv), x = it - rb * m, y0 = rb * RB;
      const double* pu = u + y0 * S + x;
      double w[RB + 2][3], fv[RB];
#pragma unroll
      for (int r = 0; r < RB + 2; ++r)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) w[r][dx] = pu[(r - 1) * S + dx - 1];
#pragma unroll
      for (int r = 0; r < RB; ++r) fv[r] = f[(y0 + r) * S + x];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        if (y0 + r < m) {
          const double au = kc_sum9(st, w[r][0], w[r][1], w[r][2], w[r + 1][0], w[r + 1][1], w[r + 1][2], w[r + 2][0],
                                    w[r + 2][1], w[r + 2][2]);
          o[(y0 + r) * S + x] = kc_jacobi_pt(w[r + 1][1], fv[r], au, st.c);
        }
      }
    }
    __syncthreads();
    double* t = u; u = o; o = t;
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = t1 - t0;
}

template <int RB>
void run(int m, int threads, long long* d, St9 st) {
  const int S = m + 2;
  size_t smem = 3 * (S + 4) * S * sizeof(double);
  cudaFuncSetAttribute(k_phase<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_phase<RB><<<1, threads, smem>>>(m, 100, d, st);
  k_phase<RB><<<1, threads, smem>>>(m, 1000, d, st);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("m=%2d threads=%4d RB=%d: %6.0f cycles/phase (%s)\n", m, threads, RB, c / 1000.0,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  St9 st{};
  for (int k = 0; k < 9; ++k) st.w[k] = -0.1;
  st.w[4] = 1.0; st.center = 1.0; st.c = 0.8;
  for (int m : {15, 31, 63}) {
    for (int threads : {256, 384, 512, 1024}) {
      run<1>(m, threads, d, st);
      run<2>(m, threads, d, st);
      run<4>(m, threads, d, st);
    }
  }
  return 0;
}
