// kc_pcg.cuh — fused PCG vector kernels on the finest level (krylov.py:60-141,
// SURVEY.md §2.3 K7).  Elementwise expressions keep numpy's rounding
// (x + alpha*p with a separately rounded product, no FMA); only the dot
// products differ from OpenBLAS ddot in the last bits, so PCG
// histories match the reference to ~1e-12 relative, not bitwise.
//
// Scalars live in device memory and alpha = rz/pap, beta = rz_next/rz are
// formed per thread with the same IEEE division the reference's Python
// floats use.  Guards make the update kernels no-ops when the reference would
// have stopped for breakdown (pap <= 0 or rz_next <= 0), so the host can
// inspect the scalars after the fact without the device having run ahead.
#pragma once
#include "kc_common.cuh"
#include "kc_grid_kernels.cuh"

// r = f - A x (krylov.py:76).  Grid-stride over rows like the reductions.
__global__ void __launch_bounds__(KC_RED_THREADS)
    k_pcg_residual(const double* __restrict__ x, const double* __restrict__ f, double* __restrict__ r, int m,
                   int P, St9 s) {
  for (int y = blockIdx.x; y < m; y += gridDim.x)
    for (int xx = threadIdx.x; xx < m; xx += KC_RED_THREADS) {
      const size_t i = kc_idx(P, y, xx);
      r[i] = DSUB(__ldg(f + i), kc_apply9(x + i, P, s));
    }
}

// ap = A p ; partial[block] = sum p*ap (krylov.py:109-110).  A thread owns
// one column and slides a 3x3 register window down KC_RY rows (3 new loads
// per row instead of 9), like k_jacobi; blocks of KC_BX x KC_BY threads,
// one deterministic partial per block.
#define KC_PCG_BLOCKS(m) (((m) + KC_BX - 1) / KC_BX * (((m) + KC_BY * KC_RY - 1) / (KC_BY * KC_RY)))
__global__ void __launch_bounds__(KC_BX* KC_BY)
    k_pcg_apply_dot(const double* __restrict__ p, double* __restrict__ ap, int m, int P, St9 s,
                    double* __restrict__ part) {
  const int x = blockIdx.x * KC_BX + threadIdx.x;
  const int y0 = (blockIdx.y * KC_BY + threadIdx.y) * KC_RY;
  double acc = 0.0;
  if (x < m && y0 < m) {
    const double* pu = p + kc_idx(P, y0, x);
    double a0 = __ldg(pu - P - 1), a1 = __ldg(pu - P), a2 = __ldg(pu - P + 1);
    double b0 = __ldg(pu - 1), b1 = __ldg(pu), b2 = __ldg(pu + 1);
#pragma unroll
    for (int k = 0; k < KC_RY; ++k) {
      if (y0 + k >= m) break;
      const double* pn = pu + (size_t)(k + 1) * P;
      const double c0 = __ldg(pn - 1), c1 = __ldg(pn), c2 = __ldg(pn + 1);
      const double a = kc_sum9(s, a0, a1, a2, b0, b1, b2, c0, c1, c2);
      ap[kc_idx(P, y0 + k, x)] = a;
      acc = fma(b1, a, acc);
      a0 = b0; a1 = b1; a2 = b2;
      b0 = c0; b1 = c1; b2 = c2;
    }
  }
  // block tree: warps, then warp 0
  __shared__ double sh[KC_BX * KC_BY / 32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  const int t = threadIdx.y * KC_BX + threadIdx.x;
  if ((t & 31) == 0) sh[t >> 5] = acc;
  __syncthreads();
  if (t == 0) {
    double b = 0.0;
    for (int w = 0; w < KC_BX * KC_BY / 32; ++w) b += sh[w];
    part[blockIdx.y * gridDim.x + blockIdx.x] = b;
  }
}

// The same with two columns per thread: one 16-byte load of the row pair
// plus its two outer neighbours per row (3 loads per 2 outputs instead of 3
// per output; the one-column kernel reached ~0.53 of HBM peak, ncu host-loop
// capture, tools/ncu_pcg.py host).  Per-point arithmetic unchanged.
#define KC_PCG_BLOCKS2(m) (((m) + 2 * KC_BX - 1) / (2 * KC_BX) * (((m) + KC_BY * KC_RY - 1) / (KC_BY * KC_RY)))
__global__ void __launch_bounds__(KC_BX* KC_BY)
    k_pcg_apply_dot2(const double* __restrict__ p, double* __restrict__ ap, int m, int P, St9 s,
                     double* __restrict__ part) {
  const int x0 = 2 * (blockIdx.x * KC_BX + threadIdx.x);
  const int y0 = (blockIdx.y * KC_BY + threadIdx.y) * KC_RY;
  double acc = 0.0;
  if (x0 < m && y0 < m) {
    const double* pu = p + kc_idx(P, y0, x0);  // 16-byte aligned: P, KC_OX and x0 even
    auto row = [&](const double* q, double& l, double2& c, double& r) {
      c = __ldg(reinterpret_cast<const double2*>(q));
      l = __ldg(q - 1);
      r = __ldg(q + 2);
    };
    double al, ar, bl, br;
    double2 ac, bc;
    row(pu - P, al, ac, ar);
    row(pu, bl, bc, br);
    const bool two = x0 + 1 < m;
#pragma unroll
    for (int k = 0; k < KC_RY; ++k) {
      if (y0 + k >= m) break;
      double cl, cr;
      double2 cc;
      row(pu + (size_t)(k + 1) * P, cl, cc, cr);
      const double a0 = kc_sum9(s, al, ac.x, ac.y, bl, bc.x, bc.y, cl, cc.x, cc.y);
      const double a1 = kc_sum9(s, ac.x, ac.y, ar, bc.x, bc.y, br, cc.x, cc.y, cr);
      double* o = ap + kc_idx(P, y0 + k, x0);
      if (two) *reinterpret_cast<double2*>(o) = make_double2(a0, a1);
      else o[0] = a0;
      acc = fma(bc.x, a0, acc);
      if (two) acc = fma(bc.y, a1, acc);
      al = bl; ac = bc; ar = br;
      bl = cl; bc = cc; br = cr;
    }
  }
  __shared__ double sh[KC_BX * KC_BY / 32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  const int t = threadIdx.y * KC_BX + threadIdx.x;
  if ((t & 31) == 0) sh[t >> 5] = acc;
  __syncthreads();
  if (t == 0) {
    double b = 0.0;
    for (int w = 0; w < KC_BX * KC_BY / 32; ++w) b += sh[w];
    part[blockIdx.y * gridDim.x + blockIdx.x] = b;
  }
}

// p_new = z + beta p_old (krylov.py:126; beta = rz_next / rz, p unchanged
// when rz_next <= 0 -- the loop stops there) fused with Ap and p.Ap of the
// NEXT iteration (krylov.py:109-110): the stencil's p_new values around each
// output are formed from z and p_old on the fly, so p_new is written to the
// other p buffer (the graph alternates them) -- one pass over z, p_old,
// p_new, Ap instead of two (k_pcg_update_p, k_pcg_apply_dot2).  Per-point
// arithmetic unchanged.
__global__ void __launch_bounds__(KC_BX* KC_BY)
    k_pcg_update_p_apply_dot2(const double* __restrict__ z, const double* __restrict__ pold,
                              double* __restrict__ pnew, double* __restrict__ ap, int m, int P, St9 s,
                              const double* __restrict__ scal, int s_rz_next, int s_rz, double* __restrict__ part) {
  const double rzn = scal[s_rz_next];
  const bool upd = rzn > 0.0;
  const double beta = upd ? __ddiv_rn(rzn, scal[s_rz]) : 0.0;
  const int x0 = 2 * (blockIdx.x * KC_BX + threadIdx.x);
  const int y0 = (blockIdx.y * KC_BY + threadIdx.y) * KC_RY;
  double acc = 0.0;
  if (x0 < m && y0 < m) {
    const size_t o0 = kc_idx(P, y0, x0);
    auto pv = [&](double zz, double pp) { return upd ? DADD(zz, DMUL(beta, pp)) : pp; };
    auto row = [&](size_t o, double& l, double2& c, double& r) {
      const double2 zc = __ldg(reinterpret_cast<const double2*>(z + o));
      const double2 pc = __ldg(reinterpret_cast<const double2*>(pold + o));
      c = make_double2(pv(zc.x, pc.x), pv(zc.y, pc.y));
      l = pv(__ldg(z + o - 1), __ldg(pold + o - 1));
      r = pv(__ldg(z + o + 2), __ldg(pold + o + 2));
    };
    double al, ar, bl, br;
    double2 ac, bc;
    row(o0 - P, al, ac, ar);
    row(o0, bl, bc, br);
    const bool two = x0 + 1 < m;
#pragma unroll
    for (int k = 0; k < KC_RY; ++k) {
      if (y0 + k >= m) break;
      double cl, cr;
      double2 cc;
      row(o0 + (size_t)(k + 1) * P, cl, cc, cr);
      const double a0 = kc_sum9(s, al, ac.x, ac.y, bl, bc.x, bc.y, cl, cc.x, cc.y);
      const double a1 = kc_sum9(s, ac.x, ac.y, ar, bc.x, bc.y, br, cc.x, cc.y, cr);
      const size_t o = o0 + (size_t)k * P;
      if (two) {
        *reinterpret_cast<double2*>(ap + o) = make_double2(a0, a1);
        *reinterpret_cast<double2*>(pnew + o) = bc;
      } else {
        ap[o] = a0;
        pnew[o] = bc.x;
      }
      acc = fma(bc.x, a0, acc);
      if (two) acc = fma(bc.y, a1, acc);
      al = bl; ac = bc; ar = br;
      bl = cl; bc = cc; br = cr;
    }
  }
  __shared__ double sh[KC_BX * KC_BY / 32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  const int t = threadIdx.y * KC_BX + threadIdx.x;
  if ((t & 31) == 0) sh[t >> 5] = acc;
  __syncthreads();
  if (t == 0) {
    double b = 0.0;
    for (int w = 0; w < KC_BX * KC_BY / 32; ++w) b += sh[w];
    part[blockIdx.y * gridDim.x + blockIdx.x] = b;
  }
}

// Device-resident PCG loop state (kc_engine.cu get_pcg_graph): iterations
// completed, limits, outcome, history of the stopping measure.
struct PcgState {
  double target;
  int it, max_it, status, napp;
  double* hist;
};

// x += alpha p ; r -= alpha ap ; partial = sum (x^2 | r^2)  (krylov.py:114-117)
// With a loop state the update also waits for the previous iteration's
// checks to pass (rz > 0, budget left), which k_pcg_check evaluates after it.
template <bool MEASURE_X>
__global__ void __launch_bounds__(KC_RED_THREADS)
    k_pcg_update_xr(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                    const double* __restrict__ ap, int m, int P, const double* __restrict__ scal, int s_rz,
                    int s_pap, double* __restrict__ part, const PcgState* __restrict__ st) {
  const double pap = scal[s_pap];
  double acc = 0.0;
  const bool go = pap > 0.0 && (!st || (scal[s_rz] > 0.0 && st->it < st->max_it));
  if (go) {
    const double alpha = __ddiv_rn(scal[s_rz], pap);
    for (int y = blockIdx.x; y < m; y += gridDim.x)
      for (int xx = threadIdx.x; xx < m; xx += KC_RED_THREADS) {
        const size_t i = kc_idx(P, y, xx);
        const double xn = DADD(x[i], DMUL(alpha, __ldg(p + i)));
        const double rn = DSUB(r[i], DMUL(alpha, __ldg(ap + i)));
        x[i] = xn;
        r[i] = rn;
        acc = MEASURE_X ? fma(xn, xn, acc) : fma(rn, rn, acc);
      }
  }
  const double t = kc_block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// p = z + (rz_next / rz) p  (krylov.py:127)
__global__ void __launch_bounds__(KC_RED_THREADS)
    k_pcg_update_p(double* __restrict__ p, const double* __restrict__ z, int m, int P,
                   const double* __restrict__ scal, int s_rz_next, int s_rz) {
  const double rzn = scal[s_rz_next];
  if (!(rzn > 0.0)) return;
  const double beta = __ddiv_rn(rzn, scal[s_rz]);
  for (int y = blockIdx.x; y < m; y += gridDim.x)
    for (int xx = threadIdx.x; xx < m; xx += KC_RED_THREADS) {
      const size_t i = kc_idx(P, y, xx);
      p[i] = DADD(__ldg(z + i), DMUL(beta, p[i]));
    }
}

__global__ void k_copy_scalar(double* __restrict__ scal, int dst, int src) {
  if (threadIdx.x == 0) scal[dst] = scal[src];
}

// Stopping logic of one device PCG iteration (krylov.py:100-130), run after
// the x/r update: rz (from the previous preconditioning) must be positive,
// the budget not exhausted, pAp positive; then the measure is recorded and
// compared with the target.  Sets the loop condition (and the body's when
// set_body).
__global__ void k_pcg_check(cudaGraphConditionalHandle h_loop, cudaGraphConditionalHandle h_body, int set_body,
                            PcgState* __restrict__ st, const double* __restrict__ scal, int s_rz, int s_pap,
                            int s_meas) {
  if (threadIdx.x != 0) return;
  unsigned go = 0u;
  if (!(scal[s_rz] > 0.0)) {
    st->status = KC_STATUS_BREAKDOWN;
  } else if (st->it >= st->max_it) {
    st->status = KC_STATUS_MAX_CYCLES;
  } else {
    const int it = st->it + 1;
    st->it = it;
    if (!(scal[s_pap] > 0.0)) {  // no measure at this step (krylov.py:110-112)
      st->status = KC_STATUS_BREAKDOWN;
      st->hist[it] = __longlong_as_double(0x7ff8000000000000LL);  // NaN marks it
    } else {
      const double meas = scal[s_meas];
      st->hist[it] = meas;
      if (meas <= st->target) {
        st->status = KC_STATUS_CONVERGED;
      } else {
        go = 1u;
        st->napp += 1;
      }
    }
  }
  cudaGraphSetConditional(h_loop, go);
  if (set_body) cudaGraphSetConditional(h_body, go);
}
