// kc_dist.cuh — strip kernels of the distributed solvers' device-side loops
// (multi-GPU PCG and the batched stand-alone loop; distributed.py).
//
// The distributed drivers keep every scalar of the reference's loops
// (krylov.py:91-128, cycle.py:331-353) in a small device array `scal`
// (KC_DS_* slots, include/kcb200.h): per-rank partial sums are written into
// a slot, allreduced in place by the caller's communicator (NCCL), and a
// one-thread step kernel (k_dist_step) applies the reference's decision
// logic -- breakdown tests, alpha / beta, the stopping and divergence rules,
// the iteration counter and the history.  Nothing is read back by the host
// inside an iteration, so a batch of iterations is one CUDA graph replay and
// the host looks at the DONE flag once per batch.  Once DONE is set the
// vector updates of later (batched) iterations are skipped, so x, r, p keep
// the values of the iteration the loop stopped at; the stand-alone loop
// saves its iterate with k_strip_copy_if when the stop fires.
//
// Per-point arithmetic is the reference's numpy expression order
// (x + alpha*p, r - alpha*ap, z + beta*p; kc_common.cuh), the partial sums
// are fixed-order trees (deterministic per rank; the allreduce order is
// NCCL's).
#pragma once
#include "../../include/kcb200.h"
#include "kc_common.cuh"

#define KDS_NB KC_DS_PART  // blocks of the strip reductions (4 per SM)

// Ap = A p on the strip's own rows (p carries one halo row each side) and
// the partial p . Ap; skipped once the loop is done
__global__ void __launch_bounds__(256) k_strip_apply_dot(const double* __restrict__ p, double* __restrict__ ap, int ny,
                                                        int nx, int pitch, St9 s, double* __restrict__ part,
                                                        const double* __restrict__ scal) {
  if (scal && scal[KC_DS_DONE] != 0.0) return;
  double acc = 0.0;
  for (int y = blockIdx.x; y < ny; y += gridDim.x)
    for (int x = threadIdx.x; x < nx; x += 256) {
      const long long i = (long long)y * pitch + x;
      const double a = kc_apply9(p + i, pitch, s);
      ap[i] = a;
      acc = fma(p[i], a, acc);
    }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  __shared__ double sh[8];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += sh[k];
    part[blockIdx.x] = t;
  }
}

// partial a . b over the strip's own rows
__global__ void __launch_bounds__(256) k_strip_dot(const double* __restrict__ a, const double* __restrict__ b, int ny,
                                                  int nx, int pitch, double* __restrict__ part,
                                                  const double* __restrict__ scal) {
  if (scal && scal[KC_DS_DONE] != 0.0) return;
  double acc = 0.0;
  for (int y = blockIdx.x; y < ny; y += gridDim.x)
    for (int x = threadIdx.x; x < nx; x += 256) {
      const long long i = (long long)y * pitch + x;
      acc = fma(a[i], b[i], acc);
    }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  __shared__ double sh[8];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += sh[k];
    part[blockIdx.x] = t;
  }
}

// x += alpha p ; r -= alpha ap (krylov.py:114-115) ; partial of x.x or r.r
__global__ void __launch_bounds__(256) k_strip_pcg_update_xr(double* __restrict__ x, double* __restrict__ r,
                                                            const double* __restrict__ p,
                                                            const double* __restrict__ ap, int ny, int nx, int pitch,
                                                            const double* __restrict__ scal, int measure_x,
                                                            double* __restrict__ part) {
  if (scal[KC_DS_DONE] != 0.0) return;
  const double alpha = scal[KC_DS_ALPHA];
  double acc = 0.0;
  for (int y = blockIdx.x; y < ny; y += gridDim.x)
    for (int xx = threadIdx.x; xx < nx; xx += 256) {
      const long long i = (long long)y * pitch + xx;
      const double xn = DADD(x[i], DMUL(alpha, p[i]));
      const double rn = DSUB(r[i], DMUL(alpha, ap[i]));
      x[i] = xn;
      r[i] = rn;
      acc = measure_x ? fma(xn, xn, acc) : fma(rn, rn, acc);
    }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  __shared__ double sh[8];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += sh[k];
    part[blockIdx.x] = t;
  }
}

// p = z + beta p (krylov.py:125)
__global__ void __launch_bounds__(256) k_strip_pcg_update_p(double* __restrict__ p, const double* __restrict__ z,
                                                           int ny, int nx, int pitch,
                                                           const double* __restrict__ scal) {
  if (scal[KC_DS_DONE] != 0.0) return;
  const double beta = scal[KC_DS_BETA];
  for (int y = blockIdx.x; y < ny; y += gridDim.x)
    for (int x = threadIdx.x; x < nx; x += 256) {
      const long long i = (long long)y * pitch + x;
      p[i] = DADD(z[i], DMUL(beta, p[i]));
    }
}

// r = f - A x (krylov.py:76)
__global__ void __launch_bounds__(256) k_strip_residual(const double* __restrict__ x, const double* __restrict__ f,
                                                       double* __restrict__ r, int ny, int nx, int pitch, St9 s) {
  for (int y = blockIdx.x; y < ny; y += gridDim.x)
    for (int xx = threadIdx.x; xx < nx; xx += 256) {
      const long long i = (long long)y * pitch + xx;
      r[i] = DSUB(f[i], kc_apply9(x + i, pitch, s));
    }
}

// dst = src on the strip's rows when the loop stopped in the last step
__global__ void __launch_bounds__(256) k_strip_copy_if(const double* __restrict__ src, double* __restrict__ dst, int ny,
                                                      int nx, int pitch, const double* __restrict__ scal) {
  if (scal[KC_DS_JUST_DONE] == 0.0) return;
  for (int y = blockIdx.x; y < ny; y += gridDim.x)
    for (int x = threadIdx.x; x < nx; x += 256) {
      const long long i = (long long)y * pitch + x;
      dst[i] = src[i];
    }
}

// fixed-order sum of the block partials into scal[slot]
__global__ void __launch_bounds__(256) k_dist_final(const double* __restrict__ part, int nb, double* __restrict__ scal,
                                                   int slot) {
  if (scal[KC_DS_DONE] != 0.0) return;
  double t = 0.0;
  for (int b = threadIdx.x; b < nb; b += 256) t += part[b];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  __shared__ double sh[8];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int k = 0; k < 8; ++k) a += sh[k];
    scal[slot] = a;
  }
}

// The reference's scalar decisions, one step kind per point of the loop
// (slots: include/kcb200.h KC_DS_*).  hist: PCG measure history (hist[it]),
// or the stand-alone error / residual histories (hist[2 it], hist[2 it + 1]).
__global__ void k_dist_step(int kind, double* __restrict__ sc, double* __restrict__ hist) {
  if (threadIdx.x != 0) return;
  const bool was_done = sc[KC_DS_DONE] != 0.0;
  sc[KC_DS_JUST_DONE] = 0.0;
  if (was_done) return;
  auto finish = [&](int status) {
    sc[KC_DS_STATUS] = (double)status;
    sc[KC_DS_DONE] = 1.0;
    sc[KC_DS_JUST_DONE] = 1.0;
  };
  switch (kind) {
    case KC_DS_PCG_RZ0: {  // z = M r; rz = r . z (krylov.py:100-104); the caller copies p = z
      if (!(sc[KC_DS_RZN] > 0.0)) {
        finish(KC_STATUS_BREAKDOWN);
      } else {
        sc[KC_DS_RZ] = sc[KC_DS_RZN];
      }
      break;
    }
    case KC_DS_PCG_PAP: {  // iteration it: ap = A p, pap (krylov.py:107-113)
      const int it = (int)sc[KC_DS_IT] + 1;
      sc[KC_DS_IT] = (double)it;
      const double pap = sc[KC_DS_PAP];
      if (!(pap > 0.0)) {
        hist[it] = __longlong_as_double(0x7ff8000000000000LL);  // no measure at this step
        finish(KC_STATUS_BREAKDOWN);
      } else {
        sc[KC_DS_ALPHA] = __ddiv_rn(sc[KC_DS_RZ], pap);
      }
      break;
    }
    case KC_DS_PCG_MEAS: {  // after x, r updates: current = measure() (krylov.py:116-120)
      const int it = (int)sc[KC_DS_IT];
      const double cur = sqrt(sc[KC_DS_MEAS]);
      hist[it] = cur;
      if (cur <= sc[KC_DS_TARGET]) finish(KC_STATUS_CONVERGED);
      break;
    }
    case KC_DS_PCG_RZ: {  // z = M r; rz_next = r . z; beta (krylov.py:121-126)
      const double rzn = sc[KC_DS_RZN];
      if (!(rzn > 0.0)) {
        finish(KC_STATUS_BREAKDOWN);
      } else if ((int)sc[KC_DS_IT] >= (int)sc[KC_DS_MAXIT]) {
        finish(KC_STATUS_MAX_CYCLES);  // the for loop of krylov.py:106 ran out
      } else {
        sc[KC_DS_BETA] = __ddiv_rn(rzn, sc[KC_DS_RZ]);
        sc[KC_DS_RZ] = rzn;
      }
      break;
    }
    case KC_DS_SOLVE: {  // stand-alone: norms of the iterate after cycle it (cycle.py:343-353)
      const int it = (int)sc[KC_DS_IT];
      const double e = sqrt(sc[KC_DS_E2]), r = sqrt(sc[KC_DS_R2]);
      hist[2 * it] = e;
      hist[2 * it + 1] = r;
      const double cur = sc[KC_DS_STOP_RESIDUAL] != 0.0 ? r : e;
      if (it == 0) sc[KC_DS_TARGET] = cur / sc[KC_DS_REDUCTION];  // cycle.py:336-337
      if (cur <= sc[KC_DS_TARGET]) {
        finish(KC_STATUS_CONVERGED);
      } else if (it > 0) {
        const double streak = cur > sc[KC_DS_PREV] ? sc[KC_DS_STREAK] + 1.0 : 0.0;
        sc[KC_DS_STREAK] = streak;
        if (streak >= 5.0) finish(KC_STATUS_DIVERGED);
      }
      sc[KC_DS_PREV] = cur;
      if (sc[KC_DS_DONE] == 0.0) {
        if (it >= (int)sc[KC_DS_MAXIT]) finish(KC_STATUS_MAX_CYCLES);
        else sc[KC_DS_IT] = (double)(it + 1);
      }
      break;
    }
    default:
      break;
  }
}
