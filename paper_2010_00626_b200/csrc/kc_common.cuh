// kc_common.cuh — shared definitions for the B200 kappa-cycle engine.
//
// Data layout: a level with interior side m
// (= 2^(n-l+1)-1, mesh.py:63-64) is stored as (m+2) rows of P doubles:
// rows y = -1 .. m, interior x = 0 .. m-1 at column KC_OX + x, and a ghost
// ring (row -1, row m, column -1, column m) that is kept at +0.0 forever.
// The ghost ring *is* the reference's "reads outside the interior are
// implicit zeros" (mesh.py:3-5, stencil.py:108-113, transfer.py:49-52), so
// no kernel carries boundary branches.  KC_OX = 16 puts x = 0 on a 128-byte
// line; P is a multiple of 16 doubles so every row starts 128-B aligned.
// Rows also carry >= 127 columns of zero padding past the ghost column.
#pragma once
#include <cstddef>
#include <cstdint>

#define KC_OX 16

#ifndef KC_FAST
#define KC_FAST 0  // 1: the FMA-contracted build (see DADD below)
#endif

// Element (y, x) of a padded level, y, x in [-1, m].
__host__ __device__ __forceinline__ size_t kc_idx(int P, int y, int x) {
  return (size_t)(y + 1) * (size_t)P + (size_t)(KC_OX + x);
}

__host__ __device__ __forceinline__ int kc_pitch(int m) {
  // columns -1 .. m live at KC_OX-1 .. KC_OX+m; the streaming kernels read
  // 128-column bands that may run up to 127 columns past m (masked), so rows
  // carry that much zero padding
  int need = KC_OX + m + 128;
  return (need + 15) & ~15;
}

// One level's constant stencil: w[dy+1][dx+1] weights u(y+dy, x+dx)
// (stencil.py:66-70).  Taps with |w| <= DBL_EPSILON are stored as +0.0,
// which for finite data is bit-identical to scipy.ndimage.correlate skipping
// them.  c = omega / center, the scalar of
// damped_jacobi_sweep (smoother.py:95-100), computed on the host exactly as
// the reference's Python float division does.
struct St9 {
  double w[9];
  double c;
  double center;
};

// Exact (non-contracted) fp64 arithmetic.  Every stencil expression in this
// engine evaluates the reference's numpy expression in the same order with
// separately rounded multiplies and adds, so iterates are
// bit-identical to the fp64 CPU reference.
//
// KC_FAST (the second build, libkcb200_fast.so): the same expressions with
// plain operators, so nvcc contracts every a*b + c into one DFMA (a 9-point
// sum becomes 1 multiply + 8 FMAs instead of 9 multiplies + 8 adds, a Jacobi
// point update 11 fp64 instructions instead of 20).  Iterates then differ
// from the reference in the last bits; the parity bar for this build is the
// north star's (per-cycle histories within 1e-10 relative, identical
// iteration counts; tests/test_gpu_fast.py).
#if KC_FAST
#define DADD(a, b) ((a) + (b))
#define DSUB(a, b) ((a) - (b))
#define DMUL(a, b) ((a) * (b))
#define DMUL0(a, b) ((a) * (b))
#else
#define DADD(a, b) __dadd_rn((a), (b))
#define DSUB(a, b) __dsub_rn((a), (b))
#define DMUL(a, b) __dmul_rn((a), (b))
// 0.0 + a*b with the product rounded first, as one instruction: fma rounds
// the exact a*b + 0.0 once, which equals the rounded product for every
// nonzero result, and -0 + +0 = +0 covers the zero case -- bit-identical to
// DADD(0.0, DMUL(a, b)), one fp64 issue instead of two.
#define DMUL0(a, b) __fma_rn((a), (b), 0.0)
#endif

// 9-point correlation at p (pointer to u(y,x)), rows at p -/+ S.
// Accumulation order = scipy.ndimage.correlate's C order: acc = 0, then
// dy = -1..1 outer, dx = -1..1 inner (stencil.py:113).
template <typename T>
__device__ __forceinline__ double kc_apply9(const T* __restrict__ p, int S, const St9& s) {
  const T* ps = p - S;
  const T* pn = p + S;
  double acc = DMUL0(s.w[0], ps[-1]);  // 0.0 + w0 u
  acc = DADD(acc, DMUL(s.w[1], ps[0]));
  acc = DADD(acc, DMUL(s.w[2], ps[1]));
  acc = DADD(acc, DMUL(s.w[3], p[-1]));
  acc = DADD(acc, DMUL(s.w[4], p[0]));
  acc = DADD(acc, DMUL(s.w[5], p[1]));
  acc = DADD(acc, DMUL(s.w[6], pn[-1]));
  acc = DADD(acc, DMUL(s.w[7], pn[0]));
  acc = DADD(acc, DMUL(s.w[8], pn[1]));
  return acc;
}

// Same sum from nine register values (a = south row, b = centre row, c = north row).
__device__ __forceinline__ double kc_sum9(const St9& s, double a0, double a1, double a2, double b0,
                                          double b1, double b2, double c0, double c1, double c2) {
  double acc = DMUL0(s.w[0], a0);  // 0.0 + w0 a0
  acc = DADD(acc, DMUL(s.w[1], a1));
  acc = DADD(acc, DMUL(s.w[2], a2));
  acc = DADD(acc, DMUL(s.w[3], b0));
  acc = DADD(acc, DMUL(s.w[4], b1));
  acc = DADD(acc, DMUL(s.w[5], b2));
  acc = DADD(acc, DMUL(s.w[6], c0));
  acc = DADD(acc, DMUL(s.w[7], c1));
  acc = DADD(acc, DMUL(s.w[8], c2));
  return acc;
}

// Damped Jacobi point update u + (omega/center) * (f - Au) (smoother.py:100).
__device__ __forceinline__ double kc_jacobi_pt(double u, double f, double au, double c) {
  return DADD(u, DMUL(c, DSUB(f, au)));
}

// First sweep on an all-zero guess: A*0 == +0 exactly, f - (+0) == f, so the
// update is 0.0 + c*f (the +0.0 add keeps the sign of zero identical).
__device__ __forceinline__ double kc_jacobi_zero(double f, double c) {
  return DMUL0(c, f);
}

// Full weighting (transfer.py:78-83): numpy evaluates
//   ((4*C + 2*(((S + N) + W) + E)) + (((SW + SE) + NW) + NE)) / 16
// where S/N are fine rows 2q/2q+2 and W/E columns 2p/2p+2.  Division by 16
// is an exact power-of-two scaling, identical to multiplying by 0.0625.
__device__ __forceinline__ double kc_fw(double sw, double s, double se, double w, double c, double e,
                                        double nw, double n, double ne) {
  double edge = DADD(DADD(DADD(s, n), w), e);
  double corner = DADD(DADD(DADD(sw, se), nw), ne);
  return DMUL(DADD(DADD(DMUL(4.0, c), DMUL(2.0, edge)), corner), 0.0625);
}

// Bilinear prolongation value at fine (y, x) from the padded coarse array
// (transfer.py:53-57); cp(q, p) must accept q, p in [-1, mc].
template <typename F>
__device__ __forceinline__ double kc_prolong_val(int y, int x, F cp) {
  const int q = y >> 1, p = x >> 1;
  if (y & 1) {
    if (x & 1) return cp(q, p);                                   // fine[1::2, 1::2]
    return DMUL(0.5, DADD(cp(q, p - 1), cp(q, p)));               // fine[1::2, 0::2]
  }
  if (x & 1) return DMUL(0.5, DADD(cp(q - 1, p), cp(q, p)));      // fine[0::2, 1::2]
  return DMUL(0.25, DADD(DADD(DADD(cp(q - 1, p - 1), cp(q - 1, p)), cp(q, p - 1)), cp(q, p)));
}
