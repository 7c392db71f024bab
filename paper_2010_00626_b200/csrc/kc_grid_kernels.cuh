// kc_grid_kernels.cuh — whole-GPU stencil kernels for one level in HBM.
//
// Each kernel reproduces one reference operation bit-for-bit:
//   k_jacobi          damped_jacobi_sweep          smoother.py:95-100
//   k_resid_restrict  residual + restrict (full)   stencil.py:116-120, transfer.py:75-83
//   k_prolong_add     v += prolong(vc) (full)      cycle.py:174-176, transfer.py:50-58
//   k_coarsest        f / center                   cycle.py:182-190
// The hot-loop sizes (4095^2, 16383^2) are HBM-bound: a thread owns one
// column and slides a 3-row register window down KC_RY rows, so u is fetched
// from DRAM once and re-read from L1/L2 for the neighbouring taps.
#pragma once
#include "kc_common.cuh"

#define KC_BX 32
#define KC_BY 8
#define KC_RY 8

template <bool ZERO_U>
__global__ void __launch_bounds__(KC_BX* KC_BY)
    k_jacobi(const double* __restrict__ u, const double* __restrict__ f, double* __restrict__ out,
             int m, int nx, int P, St9 s) {  // m rows, nx columns
  const int x = blockIdx.x * KC_BX + threadIdx.x;
  const int y0 = (blockIdx.y * KC_BY + threadIdx.y) * KC_RY;
  if (x >= nx || y0 >= m) return;
  const size_t i0 = kc_idx(P, y0, x);
  if (ZERO_U) {
#pragma unroll
    for (int k = 0; k < KC_RY; ++k) {
      if (y0 + k >= m) break;
      const size_t i = i0 + (size_t)k * P;
      out[i] = kc_jacobi_zero(__ldg(f + i), s.c);
    }
    return;
  }
  const double* pu = u + i0;
  double a0 = __ldg(pu - P - 1), a1 = __ldg(pu - P), a2 = __ldg(pu - P + 1);
  double b0 = __ldg(pu - 1), b1 = __ldg(pu), b2 = __ldg(pu + 1);
#pragma unroll
  for (int k = 0; k < KC_RY; ++k) {
    if (y0 + k >= m) break;
    const double* pn = pu + (size_t)(k + 1) * P;
    const double c0 = __ldg(pn - 1), c1 = __ldg(pn), c2 = __ldg(pn + 1);
    const size_t i = i0 + (size_t)k * P;
    const double au = kc_sum9(s, a0, a1, a2, b0, b1, b2, c0, c1, c2);
    out[i] = kc_jacobi_pt(b1, __ldg(f + i), au, s.c);
    a0 = b0; a1 = b1; a2 = b2;
    b0 = c0; b1 = c1; b2 = c2;
  }
}

// fc(q,p) = FW(f - A u) around fine (2q+1, 2p+1).  One thread per coarse
// node; the 3x3 fine residuals are formed from a 5x5 patch of u.  ZERO_U: u is
// the all-zero guess, so r = f - (+0) = f exactly.
template <bool ZERO_U>
__global__ void __launch_bounds__(KC_BX* KC_BY)
    k_resid_restrict(const double* __restrict__ u, const double* __restrict__ f,
                     double* __restrict__ fc, int mc, int mcx, int P, int Pc, St9 s) {  // mc x mcx coarse
  const int p = blockIdx.x * KC_BX + threadIdx.x;
  const int q = blockIdx.y * KC_BY + threadIdx.y;
  if (p >= mcx || q >= mc) return;
  const int y = 2 * q + 1, x = 2 * p + 1;
  double r[3][3];
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy) {
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
      const size_t i = kc_idx(P, y + dy, x + dx);
      const double fv = __ldg(f + i);
      if (ZERO_U) {
        r[dy + 1][dx + 1] = fv;
      } else {
        r[dy + 1][dx + 1] = DSUB(fv, kc_apply9(u + i, P, s));
      }
    }
  }
  fc[kc_idx(Pc, q, p)] =
      kc_fw(r[0][0], r[0][1], r[0][2], r[1][0], r[1][1], r[1][2], r[2][0], r[2][1], r[2][2]);
}

// v += P vc (in place).  V_ZERO: v is the all-zero guess -> v = 0.0 + e.
template <bool V_ZERO>
__global__ void __launch_bounds__(KC_BX* KC_BY)
    k_prolong_add(double* __restrict__ v, const double* __restrict__ vc, int m, int nx, int P, int Pc) {
  const int x = blockIdx.x * KC_BX + threadIdx.x;
  const int y = blockIdx.y * KC_BY + threadIdx.y;
  if (x >= nx || y >= m) return;
  auto cp = [&](int q, int p) { return __ldg(vc + kc_idx(Pc, q, p)); };
  const double e = kc_prolong_val(y, x, cp);
  const size_t i = kc_idx(P, y, x);
  v[i] = DADD(V_ZERO ? 0.0 : v[i], e);
}

// out = A u (stencil.py:108-113) or f - A u (stencil.py:116-120)
template <bool RES>
__global__ void __launch_bounds__(KC_BX* KC_BY)
    k_apply(const double* __restrict__ u, const double* __restrict__ f, double* __restrict__ out, int m, int nx,
            int P, St9 s) {
  const int x = blockIdx.x * KC_BX + threadIdx.x;
  const int y = blockIdx.y * KC_BY + threadIdx.y;
  if (x >= nx || y >= m) return;
  const size_t i = kc_idx(P, y, x);
  const double a = kc_apply9(u + i, P, s);
  out[i] = RES ? DSUB(__ldg(f + i), a) : a;
}

__global__ void k_coarsest(double* __restrict__ v, const double* __restrict__ f, int P, double center) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const size_t i = kc_idx(P, 0, 0);
    v[i] = __ddiv_rn(f[i], center);
  }
}

// Zero the interior of a level (ghost ring is already zero).
__global__ void k_zero(double* __restrict__ v, int m, int nx, int P) {
  const int x = blockIdx.x * KC_BX + threadIdx.x;
  const int y = blockIdx.y * KC_BY + threadIdx.y;
  if (x >= nx || y >= m) return;
  v[kc_idx(P, y, x)] = 0.0;
}

// ---------------------------------------------------------------------------
// Deterministic fp64 reductions (mesh.py:93-102).  A fixed grid of
// KC_RED_BLOCKS blocks strides over rows in a fixed pattern; each block
// reduces in a fixed tree; a single block then sums the partials in a fixed
// tree.  No atomics: results are bit-identical run to run.
// ---------------------------------------------------------------------------
#define KC_RED_BLOCKS 592
#define KC_RED_THREADS 256

__device__ __forceinline__ double kc_block_sum(double v) {
  __shared__ double sh[KC_RED_THREADS / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < (KC_RED_THREADS / 32) ? sh[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  }
  __syncthreads();
  return t;  // valid in thread 0
}

// kind 0: sum a*b ; kind 1: sum (f - A a)^2 (b = f)
template <int KIND>
__global__ void __launch_bounds__(KC_RED_THREADS)
    k_red_partial(const double* __restrict__ a, const double* __restrict__ b, int m, int nx, int P, St9 s,
                  double* __restrict__ part) {
  double acc = 0.0;
  for (int y = blockIdx.x; y < m; y += gridDim.x) {
    for (int x = threadIdx.x; x < nx; x += KC_RED_THREADS) {
      const size_t i = kc_idx(P, y, x);
      if (KIND == 0) {
        acc = fma(__ldg(a + i), __ldg(b + i), acc);
      } else {
        const double r = DSUB(__ldg(b + i), kc_apply9(a + i, P, s));
        acc = fma(r, r, acc);
      }
    }
  }
  const double t = kc_block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// out[0] = sum(part[0..np)); if SQRT also out[0] = sqrt(sum)
template <bool SQRT>
__global__ void __launch_bounds__(KC_RED_THREADS) k_red_final(const double* __restrict__ part, int np,
                                                             double* __restrict__ out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += KC_RED_THREADS) acc += part[i];
  const double t = kc_block_sum(acc);
  if (threadIdx.x == 0) out[0] = SQRT ? sqrt(t) : t;
}
