// kc_zebra.cuh — zebra line relaxation, y-semi-coarsening transfers and the
// single-line coarsest solve (the paper's solvers 3-6).
//
//   k_zebra_rhs_x / _y   rhs = f - (cross-line part of A) u on the lines of one
//                        parity, written over those lines of u
//                        (smoother.py:119-133: woff = A with its line row /
//                        column zeroed; ndimage C-order taps, F2/F3)
//   k_zebra_solve_x / _y the constant-coefficient tridiagonal solve of every
//                        line of that parity, in place: LAPACK dgtsv (what
//                        scipy.linalg.solve_banded((1,1)) calls) restated with
//                        its elimination plan precomputed on the host
//                        (kc_engine.cu zebra_plan), so each line only replays
//                        the data-dependent right-hand-side operations
//   k_resid_restrict_semi  fc = 0.25 (r_S + 2 r_C + r_N)      transfer.py:84-86
//   k_prolong_add_semi     v += linear-in-y interpolation     transfer.py:59-66
//   k_coarsest_line        Thomas on the single coarsest line smoother.py:71-92
//
// Line ordering follows the reference: even lines (0, 2, ...) first with the
// pre-sweep odd lines, then odd lines with the updated even lines
// (smoother.py:128-133); y-lines are x-lines of the transposed arrays
// (smoother.py:111-112), so their cross-line taps accumulate in the
// transposed C order (x offset outer, y offset inner).  Every expression keeps
// the reference's operand order without FMA, so results are bit-identical.
#pragma once
#include "kc_common.cuh"

// dgtsv elimination plan of one constant-coefficient system of order n:
//   fact[n-1], piv[n-1] (row interchange at step i), and the factored
//   d[n], du[n-1], dl[n-2] (second superdiagonal, nonzero only after swaps)
struct ZPlan {
  const double* fact;
  const double* d;
  const double* du;
  const double* dl;
  const unsigned char* piv;
  int n;
  const double* rd;  // 1 / d (the FMA build's back substitution multiplies)
};

// one back-substitution quotient: the exact build divides (dgtsv's
// B(i) / D(i), correctly rounded); the FMA build multiplies by the
// precomputed reciprocal (a ~100-cycle dependent division per line step
// becomes one multiply; last-bit differences, tolerance parity)
__device__ __forceinline__ double kz_quot(double x, const ZPlan& pl, int i) {
#if KC_FAST
  return DMUL(x, __ldg(pl.rd + i));
#else
  return __ddiv_rn(x, __ldg(pl.d + i));
#endif
}

// rhs of the x-lines y = par, par + 2, ...: f - sum over rows y-1, y+1 (C order)
__global__ void k_zebra_rhs_x(double* __restrict__ u, const double* __restrict__ f, int ny, int nx, int P, St9 off,
                              int par) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = par + 2 * (blockIdx.y * blockDim.y + threadIdx.y);
  if (x >= nx || y >= ny) return;
  const size_t i = kc_idx(P, y, x);
  const double* p = u + i;
  // the line's own row has zero taps (skipped by the reference; a +0.0 term
  // never changes a sum that starts at +0.0), and is being overwritten here
  const double acc = kc_sum9(off, p[-P - 1], p[-P], p[-P + 1], 0.0, 0.0, 0.0, p[P - 1], p[P], p[P + 1]);
  u[i] = DSUB(__ldg(f + i), acc);
}

// rhs of the y-lines x = par, par + 2, ...: the transposed stencil's C order
__global__ void k_zebra_rhs_y(double* __restrict__ u, const double* __restrict__ f, int ny, int nx, int P, St9 offT,
                              int par) {
  const int x = par + 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= nx || y >= ny) return;
  const size_t i = kc_idx(P, y, x);
  const double* p = u + i;
  const double acc = kc_sum9(offT, p[-P - 1], p[-1], p[P - 1], 0.0, 0.0, 0.0, p[-P + 1], p[1], p[P + 1]);
  u[i] = DSUB(__ldg(f + i), acc);
}

// dgtsv on one line whose right-hand side b(i) = line[i * stride] (in place).
// A line solve is one thread's serial recurrence, and a zebra half-sweep has
// few lines (ny/2, or a handful on semi-coarsened levels), so the SMs hold
// few warps: every line value and plan entry is fetched KZ_CH steps ahead
// (software pipelining over two register chunks) instead of one dependent
// memory round trip per step.
#define KZ_CH 8
__device__ __forceinline__ void kz_gtsv_line(double* __restrict__ line, size_t stride, const ZPlan& pl) {
  const int n = pl.n;
  // ---- forward elimination over steps i = 0 .. n-2, carrying row i ----
  double cur = line[0];
  {
    double nv[2][KZ_CH], fa[2][KZ_CH];
    unsigned char pv[2][KZ_CH];
    auto fetch = [&](int buf, int i0) {
#pragma unroll
      for (int k = 0; k < KZ_CH; ++k) {
        const int i = i0 + k;
        if (i < n - 1) {
          nv[buf][k] = line[(size_t)(i + 1) * stride];
          fa[buf][k] = __ldg(pl.fact + i);
          pv[buf][k] = __ldg(pl.piv + i);
        }
      }
    };
    fetch(0, 0);
    for (int i0 = 0; i0 < n - 1; i0 += 2 * KZ_CH) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int ib = i0 + half * KZ_CH;
        if (ib >= n - 1) break;
        fetch(half ^ 1, ib + KZ_CH);  // next chunk in flight while this one is eliminated
#pragma unroll
        for (int k = 0; k < KZ_CH; ++k) {
          const int i = ib + k;
          if (i < n - 1) {
            if (!pv[half][k]) {  // B(i+1) = B(i+1) - FACT*B(i)
              line[(size_t)i * stride] = cur;
              cur = DSUB(nv[half][k], DMUL(fa[half][k], cur));
            } else {  // interchange: B(i) = B(i+1); B(i+1) = B(i) - FACT*B(i+1)
              line[(size_t)i * stride] = nv[half][k];
              cur = DSUB(cur, DMUL(fa[half][k], nv[half][k]));
            }
          }
        }
      }
    }
  }
  // ---- back substitution: B(i) = (B(i) - DU(i) B(i+1) - DL(i) B(i+2)) / D(i) ----
  double b1 = kz_quot(cur, pl, n - 1);
  line[(size_t)(n - 1) * stride] = b1;
  if (n < 2) return;
  // row n-2 was stored by the forward pass; it is re-read here
  double b0 = kz_quot(DSUB(line[(size_t)(n - 2) * stride], DMUL(__ldg(pl.du + n - 2), b1)), pl, n - 2);
  line[(size_t)(n - 2) * stride] = b0;
  {
    double bv[2][KZ_CH], dv[2][KZ_CH], uv[2][KZ_CH], lv2[2][KZ_CH];
    auto fetch = [&](int buf, int i0) {  // rows i0, i0-1, ..., i0-KZ_CH+1
#pragma unroll
      for (int k = 0; k < KZ_CH; ++k) {
        const int i = i0 - k;
        if (i >= 0) {
          bv[buf][k] = line[(size_t)i * stride];
          dv[buf][k] = __ldg((KC_FAST ? pl.rd : pl.d) + i);
          uv[buf][k] = __ldg(pl.du + i);
          lv2[buf][k] = __ldg(pl.dl + i);
        }
      }
    };
    fetch(0, n - 3);
    for (int i0 = n - 3; i0 >= 0; i0 -= 2 * KZ_CH) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int ib = i0 - half * KZ_CH;
        if (ib < 0) break;
        fetch(half ^ 1, ib - KZ_CH);
#pragma unroll
        for (int k = 0; k < KZ_CH; ++k) {
          const int i = ib - k;
          if (i >= 0) {
#if KC_FAST
            const double v = DMUL(DSUB(DSUB(bv[half][k], DMUL(uv[half][k], b0)), DMUL(lv2[half][k], b1)), dv[half][k]);
#else
            const double v = __ddiv_rn(DSUB(DSUB(bv[half][k], DMUL(uv[half][k], b0)), DMUL(lv2[half][k], b1)),
                                       dv[half][k]);
#endif
            line[(size_t)i * stride] = v;
            b1 = b0;
            b0 = v;
          }
        }
      }
    }
  }
}

__global__ void k_zebra_solve_x(double* __restrict__ u, int ny, int P, ZPlan pl, int par) {
  const int y = par + 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (y >= ny) return;
  kz_gtsv_line(u + kc_idx(P, y, 0), 1, pl);
}

__global__ void k_zebra_solve_y(double* __restrict__ u, int nx, int P, ZPlan pl, int par) {
  const int x = par + 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (x >= nx) return;
  kz_gtsv_line(u + kc_idx(P, 0, x), (size_t)P, pl);
}

// fc(q, x) = 0.25 ((r(2q) + 2 r(2q+1)) + r(2q+2)), r = f - A u (or f on a zero guess)
template <bool ZERO_U>
__global__ void k_resid_restrict_semi(const double* __restrict__ u, const double* __restrict__ f,
                                      double* __restrict__ fc, int mcy, int nx, int P, int Pc, St9 s) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= nx || q >= mcy) return;
  double r[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const size_t i = kc_idx(P, 2 * q + k, x);
    r[k] = ZERO_U ? __ldg(f + i) : DSUB(__ldg(f + i), kc_apply9(u + i, P, s));
  }
  fc[kc_idx(Pc, q, x)] = DMUL(0.25, DADD(DADD(r[0], DMUL(2.0, r[1])), r[2]));
}

// v += P vc: odd fine rows take coarse row q, even rows 0.5 (vc(q-1) + vc(q))
template <bool V_ZERO>
__global__ void k_prolong_add_semi(double* __restrict__ v, const double* __restrict__ vc, int ny, int nx, int P,
                                   int Pc) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= nx || y >= ny) return;
  const int q = y >> 1;
  const double e = (y & 1) ? __ldg(vc + kc_idx(Pc, q, x))
                           : DMUL(0.5, DADD(__ldg(vc + kc_idx(Pc, q - 1, x)), __ldg(vc + kc_idx(Pc, q, x))));
  const size_t i = kc_idx(P, y, x);
  v[i] = DADD(V_ZERO ? 0.0 : v[i], e);
}

// Thomas without pivoting on the single coarsest line (smoother.py:71-92);
// one thread, scratch cp in the other v buffer
__global__ void k_coarsest_line(double* __restrict__ v, const double* __restrict__ f, double* __restrict__ cp,
                                int nx, int P, double lo, double di, double up) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double* fr = f + kc_idx(P, 0, 0);
  double* x = v + kc_idx(P, 0, 0);
  double* c = cp + kc_idx(P, 0, 0);
  double piv = di;
  c[0] = __ddiv_rn(up, piv);
  x[0] = __ddiv_rn(fr[0], piv);  // dp
  for (int i = 1; i < nx; ++i) {
    piv = DSUB(di, DMUL(lo, c[i - 1]));
    c[i] = __ddiv_rn(up, piv);
    x[i] = __ddiv_rn(DSUB(fr[i], DMUL(lo, x[i - 1])), piv);
  }
  for (int i = nx - 2; i >= 0; --i) x[i] = DSUB(x[i], DMUL(c[i], x[i + 1]));
}
