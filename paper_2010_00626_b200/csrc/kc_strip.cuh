// kc_strip.cuh — per-op kernels on a row strip of a distributed level
// (multi-GPU row decomposition).
//
// A strip is ny local rows x nx columns addressed from its interior origin
// p(0,0) with row pitch `pitch` (doubles); the rows above (-1, -2) and below
// (ny, ny+1) are halo rows filled by the neighbour ranks, or the zero
// Dirichlet ghost rows at the domain boundary, and column -1 / nx are zero.
// Arithmetic is the reference's (kc_common.cuh), so a decomposed cycle is
// bit-identical to the single-domain one.
#pragma once
#include "kc_common.cuh"

#define KSTR_BX 32
#define KSTR_BY 8

// out = u + c (f - A u)  (zero_u: out = 0 + c f)   smoother.py:95-100
__global__ void __launch_bounds__(KSTR_BX* KSTR_BY)
    k_strip_jacobi(const double* __restrict__ u, const double* __restrict__ f, double* __restrict__ out, int ny,
                   int nx, int pitch, St9 s, int zero_u) {
  const int x = blockIdx.x * KSTR_BX + threadIdx.x;
  const int y = blockIdx.y * KSTR_BY + threadIdx.y;
  if (x >= nx || y >= ny) return;
  const long long i = (long long)y * pitch + x;
  out[i] = zero_u ? kc_jacobi_zero(f[i], s.c) : kc_jacobi_pt(u[i], f[i], kc_apply9(u + i, pitch, s), s.c);
}

// fc(q, p) = FW(f - A u) on the strip's coarse rows 0..ncy-1 (fine centre row
// 2q+1 local); needs u rows -1..2*ncy+1 and f rows 0..2*ncy.  transfer.py:75-83
__global__ void __launch_bounds__(KSTR_BX* KSTR_BY)
    k_strip_resid_restrict(const double* __restrict__ u, const double* __restrict__ f, double* __restrict__ fc,
                           int ncy, int ncx, int pitch, int pitch_c, St9 s, int zero_u) {
  const int p = blockIdx.x * KSTR_BX + threadIdx.x;
  const int q = blockIdx.y * KSTR_BY + threadIdx.y;
  if (p >= ncx || q >= ncy) return;
  double r[3][3];
#pragma unroll
  for (int dy = 0; dy < 3; ++dy)
#pragma unroll
    for (int dx = 0; dx < 3; ++dx) {
      const long long i = (long long)(2 * q + dy) * pitch + (2 * p + dx);
      r[dy][dx] = zero_u ? f[i] : DSUB(f[i], kc_apply9(u + i, pitch, s));
    }
  fc[(long long)q * pitch_c + p] = kc_fw(r[0][0], r[0][1], r[0][2], r[1][0], r[1][1], r[1][2], r[2][0], r[2][1], r[2][2]);
}

// v += P vc on the strip (fine local row y <-> coarse local rows (y>>1)-1 .. y>>1;
// the strip's first fine row is even)  transfer.py:50-58, cycle.py:174-176
__global__ void __launch_bounds__(KSTR_BX* KSTR_BY)
    k_strip_prolong_add(double* __restrict__ v, const double* __restrict__ vc, int ny, int nx, int pitch, int pitch_c,
                        int v_zero) {
  const int x = blockIdx.x * KSTR_BX + threadIdx.x;
  const int y = blockIdx.y * KSTR_BY + threadIdx.y;
  if (x >= nx || y >= ny) return;
  auto cp = [&](int q, int pc) { return vc[(long long)q * pitch_c + pc]; };
  const long long i = (long long)y * pitch + x;
  v[i] = DADD(v_zero ? 0.0 : v[i], kc_prolong_val(y, x, cp));
}

// partial sums over the strip's own rows: out[0] = sum a^2, out[1] = sum (f - A a)^2
__global__ void __launch_bounds__(256) k_strip_norms(const double* __restrict__ a, const double* __restrict__ f, int ny,
                                                    int nx, int pitch, St9 s, double* __restrict__ part) {
  double e = 0.0, r = 0.0;
  for (int y = blockIdx.x; y < ny; y += gridDim.x)
    for (int x = threadIdx.x; x < nx; x += 256) {
      const long long i = (long long)y * pitch + x;
      const double av = a[i];
      const double rv = DSUB(f[i], kc_apply9(a + i, pitch, s));
      e = fma(av, av, e);
      r = fma(rv, rv, r);
    }
  __shared__ double sh[2][8];
  for (int o = 16; o > 0; o >>= 1) {
    e += __shfl_down_sync(0xffffffffu, e, o);
    r += __shfl_down_sync(0xffffffffu, r, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sh[0][threadIdx.x >> 5] = e;
    sh[1][threadIdx.x >> 5] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double te = 0.0, tr = 0.0;
    for (int k = 0; k < 8; ++k) {
      te += sh[0][k];
      tr += sh[1][k];
    }
    part[2 * blockIdx.x] = te;
    part[2 * blockIdx.x + 1] = tr;
  }
}

__global__ void __launch_bounds__(256) k_strip_norms_final(const double* __restrict__ part, int nb,
                                                          double* __restrict__ out) {
  // fixed-order tree over the block partials (deterministic)
  double e = 0.0, r = 0.0;
  for (int b = threadIdx.x; b < nb; b += 256) {
    e += part[2 * b];
    r += part[2 * b + 1];
  }
  __shared__ double sh[2][8];
  for (int o = 16; o > 0; o >>= 1) {
    e += __shfl_down_sync(0xffffffffu, e, o);
    r += __shfl_down_sync(0xffffffffu, r, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sh[0][threadIdx.x >> 5] = e;
    sh[1][threadIdx.x >> 5] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double te = 0.0, tr = 0.0;
    for (int k = 0; k < 8; ++k) {
      te += sh[0][k];
      tr += sh[1][k];
    }
    out[0] = te;
    out[1] = tr;
  }
}
