// issue cost of independent 64-bit shuffles and FSEL-heavy gathers on one warp
#include <cstdio>
__global__ void k(double* out, long long* t, double a) {
  double v[16];
  for (int i = 0; i < 16; ++i) v[i] = a + i + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 64; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __shfl_sync(0xffffffffu, v[i], (threadIdx.x + 1 + (i & 1)) & 31);
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 16; ++i) s += v[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) t[0] = t1 - t0;
}
int main() {
  double* o; long long* t; cudaMalloc(&o, 256 * 8); cudaMallocManaged(&t, 64);
  for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(o, t, 1.0); cudaDeviceSynchronize(); }
  printf("16 independent 64-bit shuffles: %.1f cycles per batch (%.2f cyc per SHFL instr)\n", t[0] / 64.0, t[0] / 64.0 / 32);
}
