// kc_stream.cuh — fused streaming kernels for the HBM-resident levels.
//
//   k_pre<NU, ZERO>        NU damped-Jacobi sweeps + residual + full-weighting
//                          restriction in one pass (SURVEY.md §2.3 K1+K2+K8):
//                          reads v, f; writes v' and the coarse f.
//   k_post<NU, VZ, NORMS>  v + P vc, then NU sweeps (K3+K1), optionally with
//                          ||v'||^2 and ||f - A v'||^2 partial sums fused in
//                          (the stand-alone stopping test, cycle.py:345).
//
// Each warp streams down a band of 64 fine columns (2 per lane), one input
// row per step.  Stage t (t = 1..D) takes the row stage t-1 produced in the
// same step and completes its own row yin - t: the 9-point sum of an output
// row is accumulated over the three steps that deliver its south, centre and
// north input rows (ks_step; the reference's C order is kept), so each row
// is shuffled once for its x-neighbours and the dependent chain per stage
// and step is three taps plus the update.  Every stage loses one column of
// validity per side, so a band owns NPB coarse columns (2*NPB fine columns)
// and recomputes a thin halo; rows stream without recomputation apart from a
// short warm-up per chunk, and the chunks are sized so all warps of a launch
// form one wave (kc_engine.cu ks_choose_nq).  Loads of rows outside [-1, m]
// are clamped onto the all-zero ghost rows, so the hot loop has no branches.
//
// Per-point arithmetic is the reference's (kc_common.cuh), bit-identical to
// the per-op kernels and to scipy/numpy.  Points outside the interior are
// forced to +0.0 at every stage (the Dirichlet ghost values).
#pragma once
#include "kc_common.cuh"
#include "kc_loop.cuh"

#define KS_BAND 64  // fine columns per warp band (2 per lane)
#ifndef KS_MINB
#define KS_MINB 4   // __launch_bounds__ min blocks per SM of the streaming kernels
#endif
#ifndef KS_UNROLL
#define KS_UNROLL 4  // row-step unroll of k_pre's loop (1 -> 4: level-1 pre 125 -> 116 us)
#endif
#ifndef KS_UNROLL_POST
#define KS_UNROLL_POST 2  // row-step unroll of k_post's loop (3+ spills the norms variant)
#endif

struct StreamParams {
  const double* u;   // input v (current buffer); unused on a zero guess
  const double* f;   // level f
  double* uo;        // output v (the other buffer)
  double* fc;        // PRE: coarse f (output)
  const double* vc;  // POST: coarse v (input)
  int m, P, mc, Pc;
  int nbands, nq;    // bands across x; coarse rows per chunk
  St9 s;
  double* part;      // POST+NORMS: 2 partial sums per warp
  // row geometry: a whole level (rows = mg = m, gy0 = 0, hb = hbc = 1,
  // mcr = mc), or a row strip of a distributed level (multi-GPU): `rows`
  // local fine rows starting at global row gy0 (even) of mg, with hb valid
  // halo rows above and below in the buffer; mcr local coarse rows with hbc
  // coarse halo rows.  Masks use global rows, memory stays in the buffer.
  int rows, gy0, mg, hb, mcr, hbc;
  // strips: the chunks cover coarse-row positions [qlo, qhi) only (a window:
  // the interior rows a pass can compute while the halo exchange is in
  // flight, or the boundary rows after it; whole strip: 0, mcr + 1)
  int qlo, qhi;
};

__device__ __forceinline__ double kc_shfl_up1(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double kc_shfl_dn1(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }

// per-warp partial sums (a, b) -> part[2 wg], part[2 wg + 1]
__device__ __forceinline__ void ks_warp_partials(double a, double b, double* __restrict__ part, int wg, int lane) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  if (lane == 0) {
    part[2 * wg] = a;
    part[2 * wg + 1] = b;
  }
}

// Left halo HL >= D+1 (even) and the coarse columns owned per 64-column band.
template <int D>
struct KsGeom {
  static constexpr int HL = 2 * ((D + 2) / 2);
  static constexpr int NPB = (KS_BAND - 1 - D - HL) / 2;
};

__device__ __forceinline__ double2 ks_ld2(const double* __restrict__ a, size_t i) {
  return __ldg(reinterpret_cast<const double2*>(a + i));
}

// Input rows stream through per-warp shared-memory rings filled with
// cp.async (LDGSTS): each lane copies and later reads back only its own 16
// bytes, so no warp synchronisation is needed, and a load in flight never
// holds a register (a register queue would make every shift wait for it).
#ifndef KS_PF
#define KS_PF 4       // prefetch distance (rows); 3 / 6 / 8 measured: 6 and 8 slower (not latency-bound)
#endif
#define KS_URING (KS_PF < 8 ? 8 : 16)  // u ring slots (> KS_PF)
// f ring: stage t reads row yin - t, so rows yin - D .. yin + KS_PF are live
__host__ __device__ constexpr int ks_fring(int D) {
  return D + KS_PF + 1 <= 8 ? 8 : (D + KS_PF + 1 <= 16 ? 16 : 32);
}
__host__ __device__ constexpr int ks_warp_smem_doubles(int D) { return (KS_URING + ks_fring(D)) * KS_BAND; }
// dynamic shared memory of a 128-thread streaming block with D stages
__host__ __device__ constexpr int ks_smem_bytes(int D) { return 4 * ks_warp_smem_doubles(D) * (int)sizeof(double); }
__device__ __forceinline__ void ks_cp16(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void ks_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void ks_cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(KS_PF) : "memory"); }
__device__ __forceinline__ double2 ks_lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }

// Lag-1 stage state of the lane's two columns (x: column c0, y: c0 + 1).
// The 9-point sum of an output row runs in the reference's C order (south
// row, centre row, north row; kc_sum9), split over the three steps in which
// those input rows arrive: b holds the south taps of the row after next, c
// the south + centre taps of the next output, cen that output's own value.
// Each input row is shuffled once (its west and east neighbours), not once
// per use.
struct KsAcc {
  double2 b, c, cen;
};
// SYM: the stencil's north and south centre taps are bitwise equal (w7 ==
// w1, true of the finest level's stencil), so w7 * n and w1 * n are the same
// rounded product and each is computed once: 2 fewer multiplies per stage.
// SYM = 2: the stencil is also point-symmetric (w0 = w8, w2 = w6, w3 = w5)
// with w0 = -w2 bitwise (the finest level's rotated stencil, stencil.py:
// 97-105): every product an input value takes part in is one of cross*u,
// ns*u, ew*u, c*u, so each is computed once, the west/east neighbours'
// products arrive by shuffle instead of their values, and w0*u, w8*u are the
// exact negations of cross*u (IEEE negation is exact; x + (-y) is x - y, and
// 0 + w0*l -- DMUL0 -- is 0 - cross*l, signed zeros included): 26 fp64
// operations per step instead of 32, bit-identical.
template <int SYM = 0>
__device__ __forceinline__ void ks_step(const St9& s, KsAcc& a, double2 n, double& aux, double& auy,
                                        double2& cen) {
  if constexpr (SYM == 2) {
    const double cx = DMUL(s.w[2], n.x), cy = DMUL(s.w[2], n.y);  // w2 = w6 = -w0 = -w8
    const double sx = DMUL(s.w[1], n.x), sy = DMUL(s.w[1], n.y);  // w1 = w7
    const double ex = DMUL(s.w[3], n.x), ey = DMUL(s.w[3], n.y);  // w3 = w5
    const double cl = kc_shfl_up1(cy), el = kc_shfl_up1(ey);      // column c0 - 1
    const double cr = kc_shfl_dn1(cx), er = kc_shfl_dn1(ex);      // column c0 + 2
    aux = DSUB(DADD(DADD(a.c.x, cl), sx), cy);
    auy = DSUB(DADD(DADD(a.c.y, cx), sy), cr);
    cen = a.cen;
    a.c.x = DADD(DADD(DADD(a.b.x, el), DMUL(s.w[4], n.x)), ey);
    a.c.y = DADD(DADD(DADD(a.b.y, ex), DMUL(s.w[4], n.y)), er);
    a.b.x = DADD(DADD(DSUB(0.0, cl), sx), cy);
    a.b.y = DADD(DADD(DSUB(0.0, cx), sy), cr);
    a.cen = n;
    return;
  }
  const double l = kc_shfl_up1(n.y), e = kc_shfl_dn1(n.x);
  const double p1x = DMUL(s.w[1], n.x), p1y = DMUL(s.w[1], n.y);
  const double p7x = SYM ? p1x : DMUL(s.w[7], n.x), p7y = SYM ? p1y : DMUL(s.w[7], n.y);
  aux = DADD(DADD(DADD(a.c.x, DMUL(s.w[6], l)), p7x), DMUL(s.w[8], n.y));
  auy = DADD(DADD(DADD(a.c.y, DMUL(s.w[6], n.x)), p7y), DMUL(s.w[8], e));
  cen = a.cen;
  a.c.x = DADD(DADD(DADD(a.b.x, DMUL(s.w[3], l)), DMUL(s.w[4], n.x)), DMUL(s.w[5], n.y));
  a.c.y = DADD(DADD(DADD(a.b.y, DMUL(s.w[3], n.x)), DMUL(s.w[4], n.y)), DMUL(s.w[5], e));
  a.b.x = DADD(DADD(DMUL0(s.w[0], l), p1x), DMUL(s.w[2], n.y));
  a.b.y = DADD(DADD(DMUL0(s.w[0], n.x), p1y), DMUL(s.w[2], e));
  a.cen = n;
}
// Dirichlet: +0.0 outside the interior (global row y)
__device__ __forceinline__ void ks_mask(double2& v, int y, int mg, bool colx_in, bool coly_in) {
  const bool in = y >= 0 && y < mg;
  v.x = (in && colx_in) ? v.x : 0.0;
  v.y = (in && coly_in) ? v.y : 0.0;
}

// ---------------------------------------------------------------------------
// PRE: NU sweeps + residual + restriction.  NORMS: also ||u||^2 of the input
// and ||f - A u||^2 (the first stage's residual) as per-warp partials: the
// stand-alone stopping test of the previous cycle's result (cycle.py:345)
// at no extra stencil work.
// ---------------------------------------------------------------------------
// Stage t (1..D) consumes the row stage t-1 produced in the same step and
// completes its own output one row behind it (ks_step), so stage t emits row
// yin - t and a chunk needs only D warm-up rows per side.
template <int NU, bool ZERO, bool NORMS = false, bool STRIP = false, int SYM = 0>
__global__ void __launch_bounds__(128, KS_MINB) k_pre(const StreamParams p) {
  constexpr int D = NU + 1;
  // row geometry (StreamParams): compile-time whole-level values unless STRIP
  const int g_rows = STRIP ? p.rows : p.m, g_y0 = STRIP ? p.gy0 : 0, g_mg = STRIP ? p.mg : p.m;
  const int g_hb = STRIP ? p.hb : 1, g_mcr = STRIP ? p.mcr : p.mc;
  using G = KsGeom<D>;
  const int lane = threadIdx.x & 31;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int band = wg % p.nbands, chunk = wg / p.nbands;
  const int P0 = band * G::NPB, Q0 = (STRIP ? p.qlo : 0) + chunk * p.nq;
  const int Qe = STRIP ? min(Q0 + p.nq, p.qhi) : Q0 + p.nq;  // this chunk's coarse rows: [Q0, Qe)
  if (Q0 > g_mcr || (STRIP && Q0 >= p.qhi)) {  // whole warp
    if (NORMS) reinterpret_cast<double2*>(p.part)[wg * 32 + lane] = make_double2(0.0, 0.0);
    return;
  }
  const int m = p.m, P = p.P;
  const int XS = 2 * P0 - G::HL;
  double acc_e = 0.0, acc_r = 0.0;
  const int c0 = XS + 2 * lane;
  const bool colx_in = c0 >= 0 && c0 < m, coly_in = c0 + 1 >= 0 && c0 + 1 < m;
  const int pcol = c0 >> 1;  // coarse column of this lane (c0 even)
  const bool own_lane = lane >= G::HL / 2 && lane < G::HL / 2 + G::NPB;
  const St9 s = p.s;
  // the rows this lane writes, as half-open ranges (one unsigned compare each)
  const int ya = max(2 * Q0, 0), yb = own_lane ? min(2 * Qe, g_rows) : ya;  // uo rows
  const int qa = max(Q0, 0), qb = (own_lane && pcol < p.mc) ? min(Qe, g_mcr) : qa;  // fc rows
  auto in_rng = [](int v, int lo, int hi) { return (unsigned)(v - lo) < (unsigned)(hi - lo); };

  KsAcc A[D + 1];  // pending sums of stages 1..D
#pragma unroll
  for (int t = 0; t <= D; ++t) A[t].b = A[t].c = A[t].cen = make_double2(0.0, 0.0);
  double2 R[3] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};  // residual rows
  double RE[3] = {0.0, 0.0, 0.0};  // their values one column east of the lane's pair

  const int ys = 2 * Q0 - D;
  const int ye = 2 * Qe + D;  // inclusive: residual row 2 Qe
  // only warps touching the domain boundary need masks / row clamping
  // (a warp vote: the compiler then knows the branches on it are uniform)
  const bool edge = __any_sync(0xffffffffu, XS < 0 || XS + KS_BAND - 1 >= m || g_y0 + ys - D - 1 < 0 ||
                                                g_y0 + ye + 1 >= g_mg);
  // rows outside the buffer read its edge rows (the all-zero ghost rows of a
  // whole level): branch-free
  auto rp = [&](int y) -> size_t { return kc_idx(P, min(max(y, -g_hb), g_rows + g_hb - 1), c0); };
  // shared-memory rings (this warp's slice): u rows and f rows
  extern __shared__ double ks_smem[];
  constexpr int FR = ks_fring(D);
  double* ring = ks_smem + (threadIdx.x >> 5) * ks_warp_smem_doubles(D) + 2 * lane;
  double* uring = ring;
  double* fring = ring + KS_URING * KS_BAND;
  // one commit group per row: f(y) and, for rows the loop consumes, u(y).
  // No two copies in flight may target the same slot (their completion
  // order is not defined), hence u only from row ys on.
  auto fetch = [&](int y, bool with_u) {
    const size_t i = rp(y);
    if (!ZERO && with_u) ks_cp16(uring + (y & (KS_URING - 1)) * KS_BAND, p.u + i);
    ks_cp16(fring + (y & (FR - 1)) * KS_BAND, p.f + i);
    ks_cp_commit();
  };
  // f rows from ys-D (stage D's row in the first step) up to ys+KS_PF-1
  for (int y = ys - D; y < ys + KS_PF; ++y) fetch(y, y >= ys);
  // deeper stages, and the shared-product norms pass, spill when unrolled x4
  constexpr int UR = NU > 2 ? 1 : (SYM && NORMS && KS_UNROLL > 2) ? 2 : KS_UNROLL;
  // f of the row each stage completes (yin - t), carried in registers: stage
  // t+1's row is the one stage t had one step earlier, so a step reads one
  // new f row (yin - 1); rows ys-2 .. ys-D are loaded before the loop
  double2 fr[D + 1];
  asm volatile("cp.async.wait_group %0;" ::"n"(KS_PF + 1) : "memory");  // rows <= ys - 2 have landed
#pragma unroll
  for (int t = 1; t < D; ++t) fr[t] = ks_lds2(fring + ((ys - 1 - t) & (FR - 1)) * KS_BAND);
#pragma unroll UR
  for (int yin = ys; yin <= ye; ++yin) {
    fetch(yin + KS_PF, true);
    ks_cp_wait();  // all but the newest KS_PF groups done: rows <= yin have landed
    const double2 u0 = ZERO ? make_double2(0.0, 0.0) : ks_lds2(uring + (yin & (KS_URING - 1)) * KS_BAND);
#pragma unroll
    for (int t = D; t > 1; --t) fr[t] = fr[t - 1];
    fr[1] = ks_lds2(fring + ((yin - 1) & (FR - 1)) * KS_BAND);

    // NORMS: rows owned by this chunk, interior columns owned by this lane;
    // the input's residual is the first stage's f - A u at row yin - 1
    const int y1 = yin - 1;
    const bool own_e = NORMS && in_rng(yin, ya, yb);
    const bool own_r = NORMS && in_rng(y1, ya, yb);
    if (own_e) acc_e = fma(u0.y, u0.y, fma(u0.x, u0.x, acc_e));
    double2 nw[D + 1];
    nw[0] = u0;
    if (edge) ks_mask(nw[0], yin + g_y0, g_mg, colx_in, coly_in);  // Dirichlet: +0.0 outside the interior
#pragma unroll
    for (int t = 1; t <= D; ++t) {
      double ox, oy;
      if (ZERO && t == 1) {  // first sweep on the zero guess: 0 + c f (NU = 0: the residual is f)
        ox = NU > 0 ? kc_jacobi_zero(fr[1].x, s.c) : fr[1].x;
        oy = NU > 0 ? kc_jacobi_zero(fr[1].y, s.c) : fr[1].y;
      } else {
        double ax, ay;
        double2 cen;
        ks_step<SYM>(s, A[t], nw[t - 1], ax, ay, cen);
        const double rx = DSUB(fr[t].x, ax), ry = DSUB(fr[t].y, ay);
        if (t <= NU) {
          ox = DADD(cen.x, DMUL(s.c, rx));  // kc_jacobi_pt
          oy = DADD(cen.y, DMUL(s.c, ry));
        } else {
          ox = rx;
          oy = ry;
        }
        if (NORMS && t == 1 && own_r) acc_r = fma(colx_in ? rx : 0.0, rx, fma(coly_in ? ry : 0.0, ry, acc_r));
      }
      nw[t] = make_double2(ox, oy);
      if (edge) ks_mask(nw[t], yin - t + g_y0, g_mg, colx_in, coly_in);
    }

    // ---- restriction: residual rows yr-2, yr-1, yr (yr = yin - D, newest) --
    R[0] = R[1];
    R[1] = R[2];
    R[2] = nw[D];
    RE[0] = RE[1];
    RE[1] = RE[2];
    RE[2] = kc_shfl_dn1(nw[D].x);
    {
      const int yr = yin - D;
      const int q = (yr >> 1) - 1;
      if (!(yr & 1) && in_rng(q, qa, qb))
        p.fc[kc_idx(p.Pc, q, pcol)] = kc_fw(R[0].x, R[0].y, RE[0], R[1].x, R[1].y, RE[1], R[2].x, R[2].y, RE[2]);
    }
    // ---- output v after NU sweeps ----------------------------------------
    if (NU > 0) {
      const int y = yin - NU;
      if (in_rng(y, ya, yb)) *reinterpret_cast<double2*>(p.uo + kc_idx(P, y, c0)) = nw[NU];
    }
    // per-lane partials, stored from inside the loop: any code after it (a
    // warp reduction, even a store) makes the compiler wrap the hot loop in
    // a reconvergence region with divergence checks at every shuffle
    if (NORMS && yin == ye) reinterpret_cast<double2*>(p.part)[wg * 32 + lane] = make_double2(acc_e, acc_r);
  }
}

// ---------------------------------------------------------------------------
// POST: v + P vc, NU sweeps, optional fused norms of the result
// ---------------------------------------------------------------------------
// NM = 0: plain; 1: ||v'||^2 and ||f - A v'||^2 (one extra residual stage,
// per-warp partials); 2: f . v' (the PCG rz = r . z of a preconditioning
// cycle, whose f is r and whose result is z; per-lane partials, NU >= 1).
template <int NU, bool VZ, int NM, bool STRIP = false, int SYM = 0>
__global__ void __launch_bounds__(128, KS_MINB) k_post(const StreamParams p) {
  constexpr bool NORMS = NM == 1, DOT = NM == 2;
  const int g_rows = STRIP ? p.rows : p.m, g_y0 = STRIP ? p.gy0 : 0, g_mg = STRIP ? p.mg : p.m;
  const int g_hb = STRIP ? p.hb : 1, g_mcr = STRIP ? p.mcr : p.mc, g_hbc = STRIP ? p.hbc : 1;
  static_assert(!DOT || NU >= 1, "the f . v partials use the f row of the last sweep");
  constexpr int D = NU + (NORMS ? 1 : 0);
  constexpr int DD = D > 0 ? D : 1;
  using G = KsGeom<DD>;
  const int lane = threadIdx.x & 31;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int band = wg % p.nbands, chunk = wg / p.nbands;
  const int P0 = band * G::NPB, Q0 = (STRIP ? p.qlo : 0) + chunk * p.nq;
  const int Qe = STRIP ? min(Q0 + p.nq, p.qhi) : Q0 + p.nq;  // see k_pre
  double acc_e = 0.0, acc_r = 0.0;
  const bool active = Q0 <= g_mcr && (!STRIP || Q0 < p.qhi);
  if (DOT && !active) reinterpret_cast<double2*>(p.part)[wg * 32 + lane] = make_double2(0.0, 0.0);
  const int m = p.m, P = p.P;
  const int XS = 2 * P0 - G::HL;
  const int c0 = XS + 2 * lane;
  const bool colx_in = c0 >= 0 && c0 < m, coly_in = c0 + 1 >= 0 && c0 + 1 < m;
  const int pc = c0 >> 1;
  const bool own_lane = lane >= G::HL / 2 && lane < G::HL / 2 + G::NPB;
  const St9 s = p.s;
  const int ya = max(2 * Q0, 0), yb = own_lane ? min(2 * Qe, g_rows) : ya;  // uo rows (see k_pre)
  auto in_rng = [](int v, int lo, int hi) { return (unsigned)(v - lo) < (unsigned)(hi - lo); };

  if (active) {
    KsAcc A[DD + 1];
#pragma unroll
    for (int t = 0; t <= DD; ++t) A[t].b = A[t].c = A[t].cen = make_double2(0.0, 0.0);
    const int ys = 2 * Q0 - D;
    const int ye = 2 * Qe - 1 + D;
    const bool edge = __any_sync(0xffffffffu, XS < 0 || XS + KS_BAND - 1 >= m || g_y0 + ys - D - 2 < 0 ||
                                                  g_y0 + ye + 2 >= g_mg);
    auto rp = [&](int y) -> size_t { return kc_idx(P, min(max(y, -g_hb), g_rows + g_hb - 1), c0); };
    auto ldc = [&](int q) -> double {
      return __ldg(p.vc + kc_idx(p.Pc, min(max(q, -g_hbc), g_mcr + g_hbc - 1), pc));
    };
    // coarse rows around the input row: vcp = row q-1, vcc = row q (q = floor(yin/2))
    int qcur = ys >> 1;  // arithmetic shift: floor
    double vcp = ldc(qcur - 1), vcc = ldc(qcur), vcn = ldc(qcur + 1);
    extern __shared__ double ks_smem[];
    constexpr int FR = ks_fring(DD);
    double* ring = ks_smem + (threadIdx.x >> 5) * ks_warp_smem_doubles(DD) + 2 * lane;
    double* uring = ring;
    double* fring = ring + KS_URING * KS_BAND;
    auto fetch = [&](int y, bool with_u) {  // see k_pre: u only from row ys on
      const size_t i = rp(y);
      if (!VZ && with_u) ks_cp16(uring + (y & (KS_URING - 1)) * KS_BAND, p.u + i);
      ks_cp16(fring + (y & (FR - 1)) * KS_BAND, p.f + i);
      ks_cp_commit();
    };
    for (int y = ys - D; y < ys + KS_PF; ++y) fetch(y, y >= ys);
    constexpr int UR = (NU <= 2 || !NORMS) ? KS_UNROLL_POST : 1;  // deeper norm stages spill
    double2 fr[DD + 1];  // f of row yin - t, carried across steps (see k_pre)
    asm volatile("cp.async.wait_group %0;" ::"n"(KS_PF + 1) : "memory");
#pragma unroll
    for (int t = 1; t < D; ++t) fr[t] = ks_lds2(fring + ((ys - 1 - t) & (FR - 1)) * KS_BAND);
#pragma unroll UR
    for (int yin = ys; yin <= ye; ++yin) {
      fetch(yin + KS_PF, true);
      ks_cp_wait();
      const double2 u0 = VZ ? make_double2(0.0, 0.0) : ks_lds2(uring + (yin & (KS_URING - 1)) * KS_BAND);
#pragma unroll
      for (int t = D; t > 1; --t) fr[t] = fr[t - 1];
      if (D > 0) fr[1] = ks_lds2(fring + ((yin - 1) & (FR - 1)) * KS_BAND);
      const int q = yin >> 1;
      if (q != qcur) {  // advance the coarse window by one row (yin even); warp-uniform
        vcp = vcc;
        vcc = vcn;
        qcur = q;
        vcn = ldc(q + 1);
      }
      // prolongation + correction (transfer.py:50-58, cycle.py:174-176)
      const double lp = kc_shfl_up1(vcp), lc = kc_shfl_up1(vcc);  // coarse column pc-1
      double ex, ey;
      if (yin & 1) {  // fine row 2q+1
        ex = DMUL(0.5, DADD(lc, vcc));
        ey = vcc;
      } else {        // fine row 2q
        ex = DMUL(0.25, DADD(DADD(DADD(lp, vcp), lc), vcc));
        ey = DMUL(0.5, DADD(vcp, vcc));
      }
      double2 nw[DD + 1];
      nw[0] = make_double2(DADD(VZ ? 0.0 : u0.x, ex), DADD(VZ ? 0.0 : u0.y, ey));
      if (edge) ks_mask(nw[0], yin + g_y0, g_mg, colx_in, coly_in);
#pragma unroll
      for (int t = 1; t <= D; ++t) {
        double ax, ay;
        double2 cen;
        ks_step<SYM>(s, A[t], nw[t - 1], ax, ay, cen);
        const double rx = DSUB(fr[t].x, ax), ry = DSUB(fr[t].y, ay);
        if (t <= NU) nw[t] = make_double2(DADD(cen.x, DMUL(s.c, rx)), DADD(cen.y, DMUL(s.c, ry)));
        else nw[t] = make_double2(rx, ry);
        if (edge) ks_mask(nw[t], yin - t + g_y0, g_mg, colx_in, coly_in);
      }
      // output after NU sweeps (stage NU; NU = 0 writes the corrected v)
      {
        const int y = yin - NU;
        if (in_rng(y, ya, yb)) {
          *reinterpret_cast<double2*>(p.uo + kc_idx(P, y, c0)) = nw[NU];
          if (NORMS) acc_e = fma(nw[NU].y, nw[NU].y, fma(nw[NU].x, nw[NU].x, acc_e));
          if (DOT) acc_e = fma(fr[NU > 0 ? NU : 1].y, nw[NU].y, fma(fr[NU > 0 ? NU : 1].x, nw[NU].x, acc_e));
        }
      }
      if (NORMS) {
        const int y = yin - D;
        if (in_rng(y, ya, yb))
          acc_r = fma(nw[D].y, nw[D].y, fma(nw[D].x, nw[D].x, acc_r));
      }
      if (DOT && yin == ye) reinterpret_cast<double2*>(p.part)[wg * 32 + lane] = make_double2(acc_e, 0.0);
    }
  }
  if (NORMS) ks_warp_partials(acc_e, acc_r, p.part, wg, lane);
}

// ---------------------------------------------------------------------------
// POSTPRE: a routine call's post pass (v + P vc, NU2 sweeps; cycle.py:219-
// 220) fused with the NEXT call's pre pass on the same level (NU1 sweeps,
// residual, full weighting; cycle.py:211-213): the kappa-cycle's second
// recursive call (cycle.py:215-218) starts where the first one ended, so the
// intermediate v never leaves the chip.  Stage 0 is k_post's corrected input
// row, stages 1..NS (NS = NU2 + NU1) are sweeps, stage D = NS + 1 the
// residual, restricted as in k_pre; the chunk geometry is k_pre's.
// ---------------------------------------------------------------------------
#ifndef KS_MINB_PP
#define KS_MINB_PP 3  // six stages' pending sums need more than 128 registers
#endif
template <int NU2, int NU1, bool VZ>
__global__ void __launch_bounds__(128, KS_MINB_PP) k_postpre(const StreamParams p) {
  constexpr int NS = NU2 + NU1;
  constexpr int D = NS + 1;
  using G = KsGeom<D>;
  const int lane = threadIdx.x & 31;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int band = wg % p.nbands, chunk = wg / p.nbands;
  const int P0 = band * G::NPB, Q0 = chunk * p.nq;
  if (Q0 > p.mc) return;  // whole warp
  const int m = p.m, P = p.P;
  const int XS = 2 * P0 - G::HL;
  const int c0 = XS + 2 * lane;
  const bool colx_in = c0 >= 0 && c0 < m, coly_in = c0 + 1 >= 0 && c0 + 1 < m;
  const int pcol = c0 >> 1;  // coarse column of this lane (c0 even)
  const bool own_lane = lane >= G::HL / 2 && lane < G::HL / 2 + G::NPB;
  const St9 s = p.s;
  KsAcc A[D + 1];
#pragma unroll
  for (int t = 0; t <= D; ++t) A[t].b = A[t].c = A[t].cen = make_double2(0.0, 0.0);
  double2 R[3] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
  double RE[3] = {0.0, 0.0, 0.0};
  const int ys = 2 * Q0 - D;
  const int ye = 2 * Q0 + 2 * p.nq + D;  // inclusive: residual row 2 (Q0 + nq)
  const bool edge = __any_sync(0xffffffffu, XS < 0 || XS + KS_BAND - 1 >= m || ys - D - 2 < 0 || ye + 2 >= m);
  auto rp = [&](int y) -> size_t { return kc_idx(P, min(max(y, -1), m), c0); };
  auto ldc = [&](int q) -> double { return __ldg(p.vc + kc_idx(p.Pc, min(max(q, -1), p.mc), pcol)); };
  int qcur = ys >> 1;  // arithmetic shift: floor
  double vcp = ldc(qcur - 1), vcc = ldc(qcur), vcn = ldc(qcur + 1);
  extern __shared__ double ks_smem[];
  constexpr int FR = ks_fring(D);
  double* ring = ks_smem + (threadIdx.x >> 5) * ks_warp_smem_doubles(D) + 2 * lane;
  double* uring = ring;
  double* fring = ring + KS_URING * KS_BAND;
  auto fetch = [&](int y, bool with_u) {  // see k_pre: u only from row ys on
    const size_t i = rp(y);
    if (!VZ && with_u) ks_cp16(uring + (y & (KS_URING - 1)) * KS_BAND, p.u + i);
    ks_cp16(fring + (y & (FR - 1)) * KS_BAND, p.f + i);
    ks_cp_commit();
  };
  for (int y = ys - D; y < ys + KS_PF; ++y) fetch(y, y >= ys);
#pragma unroll 1
  for (int yin = ys; yin <= ye; ++yin) {
    fetch(yin + KS_PF, true);
    ks_cp_wait();
    const double2 u0 = VZ ? make_double2(0.0, 0.0) : ks_lds2(uring + (yin & (KS_URING - 1)) * KS_BAND);
    double2 fr[D + 1];
#pragma unroll
    for (int t = 1; t <= D; ++t) fr[t] = ks_lds2(fring + ((yin - t) & (FR - 1)) * KS_BAND);
    const int q = yin >> 1;
    if (q != qcur) {  // advance the coarse window by one row (yin even); warp-uniform
      vcp = vcc;
      vcc = vcn;
      qcur = q;
      vcn = ldc(q + 1);
    }
    // stage 0: prolongation + correction (transfer.py:50-58, cycle.py:174-176)
    const double lp = kc_shfl_up1(vcp), lc = kc_shfl_up1(vcc);
    double ex, ey;
    if (yin & 1) {
      ex = DMUL(0.5, DADD(lc, vcc));
      ey = vcc;
    } else {
      ex = DMUL(0.25, DADD(DADD(DADD(lp, vcp), lc), vcc));
      ey = DMUL(0.5, DADD(vcp, vcc));
    }
    double2 nw[D + 1];
    nw[0] = make_double2(DADD(VZ ? 0.0 : u0.x, ex), DADD(VZ ? 0.0 : u0.y, ey));
    if (edge) ks_mask(nw[0], yin, m, colx_in, coly_in);
#pragma unroll
    for (int t = 1; t <= D; ++t) {
      double ax, ay;
      double2 cen;
      ks_step<false>(s, A[t], nw[t - 1], ax, ay, cen);
      const double rx = DSUB(fr[t].x, ax), ry = DSUB(fr[t].y, ay);
      if (t <= NS) nw[t] = make_double2(DADD(cen.x, DMUL(s.c, rx)), DADD(cen.y, DMUL(s.c, ry)));
      else nw[t] = make_double2(rx, ry);
      if (edge) ks_mask(nw[t], yin - t, m, colx_in, coly_in);
    }
    // restriction of the residual rows yr-2, yr-1, yr (yr = yin - D)
    R[0] = R[1];
    R[1] = R[2];
    R[2] = nw[D];
    RE[0] = RE[1];
    RE[1] = RE[2];
    RE[2] = kc_shfl_dn1(nw[D].x);
    {
      const int yr = yin - D;
      const int qq = (yr >> 1) - 1;
      if (!(yr & 1) && own_lane && qq >= Q0 && qq < Q0 + p.nq && qq < p.mc && qq >= 0 && pcol < p.mc)
        p.fc[kc_idx(p.Pc, qq, pcol)] = kc_fw(R[0].x, R[0].y, RE[0], R[1].x, R[1].y, RE[1], R[2].x, R[2].y, RE[2]);
    }
    // v after all NS sweeps
    {
      const int y = yin - NS;
      if (own_lane && y >= 2 * Q0 && y < 2 * Q0 + 2 * p.nq && y >= 0 && y < m)
        *reinterpret_cast<double2*>(p.uo + kc_idx(P, y, c0)) = nw[NS];
    }
  }
}

// deterministic final sum of the per-warp partials: out[0] = sqrt(sum e), out[1] = sqrt(sum r)
__global__ void __launch_bounds__(256) k_norms_final(const double* __restrict__ part, int nw, double* __restrict__ out) {
  __shared__ double sh[2][8];
  double e = 0.0, r = 0.0;
  for (int i = threadIdx.x; i < nw; i += 256) {
    e += part[2 * i];
    r += part[2 * i + 1];
  }
  for (int o = 16; o > 0; o >>= 1) {
    e += __shfl_down_sync(0xffffffffu, e, o);
    r += __shfl_down_sync(0xffffffffu, r, o);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    sh[0][w] = e;
    sh[1][w] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double te = 0.0, tr = 0.0;
    for (int k = 0; k < 8; ++k) {
      te += sh[0][k];
      tr += sh[1][k];
    }
    out[0] = sqrt(te);
    out[1] = sqrt(tr);
  }
}

// Deterministic sum of n (a, b) pairs over KS_NB blocks; the last block to
// finish adds the block sums with a fixed-order tree: out = (sum a, sum b),
// square roots taken when SQRT.  (32 blocks and a one-thread serial final
// sum: ~3 us more per stand-alone iteration.)
#ifndef KS_NB
#define KS_NB 148
#endif
static_assert(KS_NB <= 256, "one block sum per thread in the final tree");
// CHECK: the last block also runs the stand-alone loop's stop test on the
// sums (kc_loop.cuh) -- one kernel less per loop iteration
template <bool SQRT, bool CHECK = false>
__global__ void __launch_bounds__(256) k_norms_lanes(const double2* __restrict__ part, int n, double2* __restrict__ bsum,
                                                     unsigned* __restrict__ counter, double* __restrict__ out,
                                                     LoopCheck ck = LoopCheck{}) {
  __shared__ double sh[2][8];
  __shared__ bool last;
  const int per = (n + KS_NB - 1) / KS_NB;
  const int i0 = blockIdx.x * per, i1 = min(n, i0 + per);
  double a = 0.0, b = 0.0;
  for (int i = i0 + threadIdx.x; i < i1; i += 256) {
    const double2 v = part[i];
    a += v.x;
    b += v.y;
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    sh[0][w] = a;
    sh[1][w] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ta = 0.0, tb = 0.0;
    for (int k = 0; k < 8; ++k) {
      ta += sh[0][k];
      tb += sh[1][k];
    }
    bsum[blockIdx.x] = make_double2(ta, tb);
    __threadfence();
    last = atomicAdd(counter, 1u) == KS_NB - 1;
  }
  __syncthreads();
  if (!last) return;  // block-uniform
  __threadfence();
  double ta = 0.0, tb = 0.0;
  if (threadIdx.x < KS_NB) {
    const double2 v = __ldcg(bsum + threadIdx.x);  // L2: written by other blocks
    ta = v.x;
    tb = v.y;
  }
  for (int o = 16; o > 0; o >>= 1) {
    ta += __shfl_down_sync(0xffffffffu, ta, o);
    tb += __shfl_down_sync(0xffffffffu, tb, o);
  }
  __syncthreads();  // sh reused
  if (lane == 0) {
    sh[0][w] = ta;
    sh[1][w] = tb;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0;
    for (int k = 0; k < 8; ++k) {
      sa += sh[0][k];
      sb += sh[1][k];
    }
    out[0] = SQRT ? sqrt(sa) : sa;
    out[1] = SQRT ? sqrt(sb) : sb;
    *counter = 0u;
    if (CHECK) kc_stop_test(ck, out[0], out[1]);
  }
}
