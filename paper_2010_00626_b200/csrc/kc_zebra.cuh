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

// ---------------------------------------------------------------------------
// FMA build: the line solves as a PARTITION method (separators), one block
// per 32 lines.  A line of n = K (s + 1) - 1 unknowns (K = 32 segments of s
// rows, separator rows k (s + 1) - 1 between them) is solved in three steps
// by the 32 threads of one lane position (one warp per segment):
//   1. each segment: y = T_s^-1 b (Thomas with precomputed factors);
//   2. the K-1 separators: a constant-coefficient tridiagonal system
//        (-a p_end) x_{j-1} + (d - a q_end - c p_0) x_j + (-c q_0) x_{j+1}
//          = b_sep - a y_last(seg j) - c y_first(seg j+1),
//      one thread per line;
//   3. each segment: x = y - x_left p - x_right q, p = T_s^-1 (a e_0) and
//      q = T_s^-1 (c e_end) the spikes of a separator on the segment.
// Algebraically dgtsv's solution (the constant line systems are diagonally
// dominant, so dgtsv never pivots on them); the operations differ, so the
// exact build keeps the serial dgtsv replay.  ~2.5 us per half-sweep at
// 4095 instead of one dependent 8k-step chain per line.
// ---------------------------------------------------------------------------
#define KZP_K 32
struct ZPart {
  const double* seg;  // cp[s], m[s], p[s], q[s] (segment Thomas factors and spikes)
  const double* red;  // rcp[K-1], rm[K-1] (separator Thomas factors)
  double a, c, ra;    // line sub / super diagonal, separator sub-diagonal (-a p_end)
  int s;              // segment length; 0: no partition plan (line too short)
};
template <bool XL>
__global__ void __launch_bounds__(KZP_K * 32) k_zebra_solve_part(double* __restrict__ u, int P, ZPart zp, int par,
                                                                int nl) {
  extern __shared__ double zsm[];
  const int s = zp.s;
  double* cp = zsm;  // 4 s segment constants
  double* mm = cp + s;
  double* pp = mm + s;
  double* qq = pp + s;
  __shared__ double yF[KZP_K][33], yL[KZP_K][33], xs[KZP_K][33];
  for (int i = threadIdx.x; i < 4 * s; i += blockDim.x) zsm[i] = __ldg(zp.seg + i);
  __syncthreads();
  const int t = threadIdx.x & 31, k = threadIdx.x >> 5;  // line within the block, segment
  const int j = blockIdx.x * 32 + t;                    // line in parity order
  const bool on = j < nl;
  const int line = par + 2 * j;
  auto at = [&](int i) -> double* { return XL ? u + kc_idx(P, line, i) : u + kc_idx(P, i, line); };
  const double a = zp.a, c = zp.c;
  const int r0 = k * (s + 1);
  // 1. y = T_s^-1 b on segment k (in place)
  if (on) {
    double z = DMUL(*at(r0), mm[0]);
    *at(r0) = z;
    for (int i = 1; i < s; ++i) {
      z = DMUL(DSUB(*at(r0 + i), DMUL(a, z)), mm[i]);
      *at(r0 + i) = z;
    }
    double y = z;  // y_{s-1} = z_{s-1}
    yL[k][t] = y;
    for (int i = s - 2; i >= 0; --i) {
      y = DSUB(*at(r0 + i), DMUL(cp[i], y));
      *at(r0 + i) = y;
    }
    yF[k][t] = y;
  }
  __syncthreads();
  // 2. the separators (warp 0: one line per lane)
  if (k == 0 && on) {
    const double* rcp = zp.red;
    const double* rm = rcp + (KZP_K - 1);
    double prev = 0.0;
    for (int q = 0; q < KZP_K - 1; ++q) {  // forward sweep, z kept in xs
      const int sep = (q + 1) * (s + 1) - 1;
      const double rhs = DSUB(DSUB(*at(sep), DMUL(a, yL[q][t])), DMUL(c, yF[q + 1][t]));
      prev = DMUL(DSUB(rhs, DMUL(zp.ra, prev)), __ldg(rm + q));
      xs[q][t] = prev;
    }
    double x = prev;
    *at((KZP_K - 1) * (s + 1) - 1) = x;
    for (int q = KZP_K - 3; q >= 0; --q) {
      x = DSUB(xs[q][t], DMUL(__ldg(rcp + q), x));
      xs[q][t] = x;
      *at((q + 1) * (s + 1) - 1) = x;
    }
  }
  __syncthreads();
  // 3. x = y - x_left p - x_right q on segment k
  if (on) {
    const double xl = k > 0 ? xs[k - 1][t] : 0.0;
    const double xr = k < KZP_K - 1 ? xs[k][t] : 0.0;
    for (int i = 0; i < s; ++i) {
      double* e = at(r0 + i);
      *e = DSUB(DSUB(*e, DMUL(xl, pp[i])), DMUL(xr, qq[i]));
    }
  }
}

// The same partition method for x-lines, whose values are contiguous along
// a line: the 32 lines of a block are 32 different rows, so a lane-per-line
// access touches 32 cache lines per instruction.  Each warp instead moves its
// segment through a shared-memory tile of 32 lines x KZP_TC columns, loaded
// and stored row by row (coalesced), and every lane runs its recurrence on
// the tile.  Same operations as k_zebra_solve_part<true>.
#define KZP_TC 16
__global__ void __launch_bounds__(KZP_K * 32) k_zebra_solve_part_x(double* __restrict__ u, int P, ZPart zp, int par,
                                                                  int nl) {
  extern __shared__ double zsm[];
  const int s = zp.s;
  double* cp = zsm;
  double* mm = cp + s;
  double* pp = mm + s;
  double* qq = pp + s;
  double* tiles = qq + s;  // KZP_K warps x 32 lines x (KZP_TC + 1)
  __shared__ double yF[KZP_K][33], yL[KZP_K][33], xs[KZP_K][33];
  for (int i = threadIdx.x; i < 4 * s; i += blockDim.x) zsm[i] = __ldg(zp.seg + i);
  __syncthreads();
  const int t = threadIdx.x & 31, k = threadIdx.x >> 5;
  const int j0 = blockIdx.x * 32;
  const int nw = min(32, nl - j0);
  const bool on = t < nw;
  double(*T)[KZP_TC + 1] = reinterpret_cast<double(*)[KZP_TC + 1]>(tiles + (size_t)k * 32 * (KZP_TC + 1));
  const double a = zp.a, c = zp.c;
  const int r0 = k * (s + 1);
  double* base = u + kc_idx(P, par + 2 * j0, r0);  // line j0's segment k
  const size_t ls = (size_t)2 * P;
  // two lines per warp instruction: lanes 0-15 line 2rr, lanes 16-31 line 2rr+1
  const int hl = t >> 4, col = t & 15;
  auto load = [&](int c0, int cnt) {
    for (int rr = 0; rr < 16; ++rr) {
      const int r = 2 * rr + hl;
      if (r < nw && col < cnt) T[r][col] = base[r * ls + c0 + col];
    }
    __syncwarp();
  };
  auto store = [&](int c0, int cnt) {
    __syncwarp();
    for (int rr = 0; rr < 16; ++rr) {
      const int r = 2 * rr + hl;
      if (r < nw && col < cnt) base[r * ls + c0 + col] = T[r][col];
    }
    __syncwarp();
  };
  // 1. y = T_s^-1 b: forward over the chunks, then backward
  double z = 0.0;
  for (int c0 = 0; c0 < s; c0 += KZP_TC) {
    const int cnt = min(KZP_TC, s - c0);
    load(c0, cnt);
    if (on)
      for (int kk = 0; kk < cnt; ++kk) {
        const int i = c0 + kk;
        z = i == 0 ? DMUL(T[t][kk], mm[0]) : DMUL(DSUB(T[t][kk], DMUL(a, z)), mm[i]);
        T[t][kk] = z;
      }
    store(c0, cnt);
  }
  double y = z;  // y_{s-1} = z_{s-1}
  if (on) yL[k][t] = y;
  for (int ctop = s - 2; ctop >= 0; ctop -= KZP_TC) {
    const int c0 = max(0, ctop - KZP_TC + 1), cnt = ctop - c0 + 1;
    load(c0, cnt);
    if (on)
      for (int kk = cnt - 1; kk >= 0; --kk) {
        y = DSUB(T[t][kk], DMUL(cp[c0 + kk], y));
        T[t][kk] = y;
      }
    store(c0, cnt);
  }
  if (on) yF[k][t] = y;
  __syncthreads();
  // 2. the separators (warp 0: one line per lane)
  if (k == 0 && on) {
    const double* rcp = zp.red;
    const double* rm = rcp + (KZP_K - 1);
    double* line = u + kc_idx(P, par + 2 * (j0 + t), 0);
    double prev = 0.0;
    for (int q = 0; q < KZP_K - 1; ++q) {
      const int sep = (q + 1) * (s + 1) - 1;
      const double rhs = DSUB(DSUB(line[sep], DMUL(a, yL[q][t])), DMUL(c, yF[q + 1][t]));
      prev = DMUL(DSUB(rhs, DMUL(zp.ra, prev)), __ldg(rm + q));
      xs[q][t] = prev;
    }
    double x = prev;
    line[(KZP_K - 1) * (s + 1) - 1] = x;
    for (int q = KZP_K - 3; q >= 0; --q) {
      x = DSUB(xs[q][t], DMUL(__ldg(rcp + q), x));
      xs[q][t] = x;
      line[(q + 1) * (s + 1) - 1] = x;
    }
  }
  __syncthreads();
  // 3. x = y - x_left p - x_right q
  const double xl = (on && k > 0) ? xs[k - 1][t] : 0.0;
  const double xr = (on && k < KZP_K - 1) ? xs[k][t] : 0.0;
  for (int c0 = 0; c0 < s; c0 += KZP_TC) {
    const int cnt = min(KZP_TC, s - c0);
    load(c0, cnt);
    if (on)
      for (int kk = 0; kk < cnt; ++kk)
        T[t][kk] = DSUB(DSUB(T[t][kk], DMUL(xl, pp[c0 + kk])), DMUL(xr, qq[c0 + kk]));
    store(c0, cnt);
  }
}

// Levels with few lines (y-semi-coarsening keeps 16383-long x-lines down to
// a single one) and the coarsest line: one block per line and KZL_K = 256
// segments, one thread each (s = (n + 1) / 256 - 1 rows), the separator
// system solved by thread 0.  `src` holds the right-hand sides (the line
// itself, or f for the coarsest solve), `u` receives the solution.
#define KZL_K 256
template <bool XL>
__global__ void __launch_bounds__(KZL_K) k_zebra_solve_line(double* __restrict__ u, const double* __restrict__ src,
                                                            int P, ZPart zp, int par) {
  extern __shared__ double zsm[];
  const int s = zp.s;
  double* cp = zsm;
  double* mm = cp + s;
  double* pp = mm + s;
  double* qq = pp + s;
  __shared__ double yF[KZL_K], yL[KZL_K], xs[KZL_K];
  for (int i = threadIdx.x; i < 4 * s; i += blockDim.x) zsm[i] = __ldg(zp.seg + i);
  __syncthreads();
  const int k = threadIdx.x;
  const int line = par + 2 * blockIdx.x;
  auto at = [&](double* b, int i) -> double* { return XL ? b + kc_idx(P, line, i) : b + kc_idx(P, i, line); };
  auto atc = [&](const double* b, int i) -> double { return XL ? b[kc_idx(P, line, i)] : b[kc_idx(P, i, line)]; };
  const double a = zp.a, c = zp.c;
  const int r0 = k * (s + 1);
  double z = DMUL(atc(src, r0), mm[0]);
  *at(u, r0) = z;
  for (int i = 1; i < s; ++i) {
    z = DMUL(DSUB(atc(src, r0 + i), DMUL(a, z)), mm[i]);
    *at(u, r0 + i) = z;
  }
  double y = z;
  yL[k] = y;
  for (int i = s - 2; i >= 0; --i) {
    y = DSUB(*at(u, r0 + i), DMUL(cp[i], y));
    *at(u, r0 + i) = y;
  }
  yF[k] = y;
  __syncthreads();
  if (k == 0) {
    const double* rcp = zp.red;
    const double* rm = rcp + (KZL_K - 1);
    double prev = 0.0;
    for (int q = 0; q < KZL_K - 1; ++q) {
      const int sep = (q + 1) * (s + 1) - 1;
      const double rhs = DSUB(DSUB(atc(src, sep), DMUL(a, yL[q])), DMUL(c, yF[q + 1]));
      prev = DMUL(DSUB(rhs, DMUL(zp.ra, prev)), __ldg(rm + q));
      xs[q] = prev;
    }
    double x = prev;
    *at(u, (KZL_K - 1) * (s + 1) - 1) = x;
    for (int q = KZL_K - 3; q >= 0; --q) {
      x = DSUB(xs[q], DMUL(__ldg(rcp + q), x));
      xs[q] = x;
      *at(u, (q + 1) * (s + 1) - 1) = x;
    }
  }
  __syncthreads();
  const double xl = k > 0 ? xs[k - 1] : 0.0;
  const double xr = k < KZL_K - 1 ? xs[k] : 0.0;
  for (int i = 0; i < s; ++i) {
    double* e = at(u, r0 + i);
    *e = DSUB(DSUB(*e, DMUL(xl, pp[i])), DMUL(xr, qq[i]));
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
