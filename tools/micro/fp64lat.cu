// dependent-chain latency of DADD / DMUL / DFMA and of a SHFL / LDS round trip (one warp)
#include <cstdio>
__global__ void k(double* out, long long* t, double a, double b) {
  __shared__ double sh[64];
  double x = a, y = b;
  sh[threadIdx.x] = a;
  __syncwarp();
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { x = __dadd_rn(x, y); x = __dadd_rn(x, y); x = __dadd_rn(x, y); x = __dadd_rn(x, y); }
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { x = __dmul_rn(x, y); x = __dmul_rn(x, y); x = __dmul_rn(x, y); x = __dmul_rn(x, y); }
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31); }
  long long t3 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { int j = (int)x & 31; x = sh[j] + 0.0; }
  long long t4 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { sh[threadIdx.x] = x; __syncwarp(); x = sh[(threadIdx.x + 1) & 31]; }
  long long t5 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4; }
}
int main() {
  double* o; long long* t; cudaMalloc(&o, 256); cudaMallocManaged(&t, 64);
  for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(o, t, 1.0, 1e-300); cudaDeviceSynchronize(); }
  printf("DADD %.1f  DMUL %.1f cyc/op (dependent)\n", t[0] / 1024.0, t[1] / 1024.0);
  printf("SHFL.64 round %.1f  LDS+DADD %.1f  STS+syncwarp+LDS %.1f cyc\n", t[2] / 256.0, t[3] / 256.0, t[4] / 256.0);
}
