// kc_tile.cuh — fused overlapped-tile kernels for the mid-size HBM levels.
//
// Same operations as k_pre / k_post (kc_stream.cuh) but for levels whose
// cost is latency, not bandwidth (sides 127 .. 511 here): a streaming warp
// spends most of its life warming up its stage pipeline there.  Instead each
// CTA stages one 2D tile plus a D-deep halo in shared memory and runs the
// stages one after another with a CTA barrier between them (halo points are
// recomputed by neighbouring tiles).  Per launch: one global load phase, D
// short compute phases, one store phase.
//
//   k_tile_pre<NU, ZERO>   NU sweeps + residual + full weighting
//   k_tile_post<NU, VZ>    v + P vc + NU sweeps
//
// Arithmetic is the reference's (kc_common.cuh): bit-identical results.
#pragma once
#include "kc_common.cuh"

#define KT_TY 16        // fine rows owned per tile (even)
#define KT_TX 32        // fine columns owned per tile (even)
#define KT_THREADS 512

struct TileParams {
  const double* u;
  const double* f;
  double* uo;
  double* fc;
  const double* vc;
  int m, P, mc, Pc;
  int tiles_x;
  St9 s;
};

// shared-memory footprint (doubles) of a tile kernel with D stencil stages
__host__ __device__ constexpr int kt_region(int D) { return (KT_TY + 1 + 2 * D) * (KT_TX + 1 + 2 * D); }
#define KT_CM 4  // coarse-patch margin (covers halos D <= 5)
#define KT_CH (KT_TY / 2 + 2 * KT_CM + 1)
#define KT_CW (KT_TX / 2 + 2 * KT_CM + 1)
__host__ __device__ constexpr int kt_smem_doubles(int D) { return 3 * kt_region(D) + KT_CH * KT_CW; }

// Stage t buffer covers rows [y0 - (D - t), y0 + TY + (D - t)] and likewise
// columns, stored with the full stage-0 stride so all stages share indexing:
// element (y, x) at (y - y0 + D) * W + (x - x0 + D), W = TX + 1 + 2D.
template <int D>
struct KtGeom {
  static constexpr int W = KT_TX + 1 + 2 * D;
  static constexpr int H = KT_TY + 1 + 2 * D;
};

template <int NU, bool ZERO>
__global__ void __launch_bounds__(KT_THREADS) k_tile_pre(const TileParams p) {
  constexpr int D = NU + 1;
  using G = KtGeom<D>;
  extern __shared__ double sm[];
  double* buf[2] = {sm, sm + G::H * G::W};
  double* fs = sm + 2 * G::H * G::W;
  const int tx = blockIdx.x % p.tiles_x, ty = blockIdx.x / p.tiles_x;
  const int y0 = ty * KT_TY, x0 = tx * KT_TX;
  const int m = p.m, P = p.P;
  const St9 s = p.s;
  // load u (stage 0) and f on the full region; outside [-1, m] read ghost zeros
  for (int i = threadIdx.x; i < G::H * G::W; i += KT_THREADS) {
    const int ry = i / G::W, rx = i - ry * G::W;
    const int y = y0 - D + ry, x = x0 - D + rx;
    const bool in = y >= 0 && y < m && x >= 0 && x < m;
    const size_t gi = kc_idx(P, min(max(y, -1), m), min(max(x, -1), m));
    fs[i] = __ldg(p.f + gi);
    buf[0][i] = (ZERO || !in) ? 0.0 : __ldg(p.u + gi);
  }
  __syncthreads();
  int cur = 0;
#pragma unroll 1
  for (int t = 1; t <= D; ++t) {
    const int h = D - t;  // halo of this stage
    const int rh = KT_TY + 1 + 2 * h, rw = KT_TX + 1 + 2 * h;
    const double* src = buf[cur];
    double* dst = buf[cur ^ 1];
    const bool zero_sweep = ZERO && t == 1;
    for (int i = threadIdx.x; i < rh * rw; i += KT_THREADS) {
      const int ry = i / rw, rx = i - ry * rw;
      const int y = y0 - h + ry, x = x0 - h + rx;
      const int k = (ry + t) * G::W + (rx + t);
      double v = 0.0;
      if (y >= 0 && y < m && x >= 0 && x < m) {
        if (t <= NU) {
          v = zero_sweep ? kc_jacobi_zero(fs[k], s.c) : kc_jacobi_pt(src[k], fs[k], kc_apply9(src + k, G::W, s), s.c);
        } else {
          v = (ZERO && NU == 0) ? fs[k] : DSUB(fs[k], kc_apply9(src + k, G::W, s));
        }
      }
      dst[k] = v;
    }
    __syncthreads();
    if (t == NU) {  // v after NU sweeps: owned points
      for (int i = threadIdx.x; i < KT_TY * KT_TX; i += KT_THREADS) {
        const int ry = i / KT_TX, rx = i - ry * KT_TX;
        const int y = y0 + ry, x = x0 + rx;
        if (y < m && x < m) p.uo[kc_idx(P, y, x)] = dst[(ry + D) * G::W + (rx + D)];
      }
    }
    cur ^= 1;
  }
  // full weighting of the residual (buffer cur) for the tile's coarse nodes
  const double* r = buf[cur];
  for (int i = threadIdx.x; i < (KT_TY / 2) * (KT_TX / 2); i += KT_THREADS) {
    const int qy = i / (KT_TX / 2), qx = i - qy * (KT_TX / 2);
    const int q = y0 / 2 + qy, pc = x0 / 2 + qx;
    if (q < p.mc && pc < p.mc) {
      const double* rc = r + (2 * qy + 1 + D) * G::W + (2 * qx + 1 + D);
      const double* rs = rc - G::W;
      const double* rn = rc + G::W;
      p.fc[kc_idx(p.Pc, q, pc)] = kc_fw(rs[-1], rs[0], rs[1], rc[-1], rc[0], rc[1], rn[-1], rn[0], rn[1]);
    }
  }
}

template <int NU, bool VZ>
__global__ void __launch_bounds__(KT_THREADS) k_tile_post(const TileParams p) {
  constexpr int D = NU > 0 ? NU : 1;
  using G = KtGeom<D>;
  extern __shared__ double sm[];
  double* buf[2] = {sm, sm + G::H * G::W};
  double* fs = sm + 2 * G::H * G::W;
  double* cs = sm + 3 * G::H * G::W;  // coarse v patch
  constexpr int CW = KT_CW;
  constexpr int CH = KT_CH;
  const int tx = blockIdx.x % p.tiles_x, ty = blockIdx.x / p.tiles_x;
  const int y0 = ty * KT_TY, x0 = tx * KT_TX;
  const int m = p.m, P = p.P;
  const St9 s = p.s;
  // coarse patch rows/cols q in [y0/2 - CM, y0/2 + TY/2 + CM], clamped onto the ghost ring
  const int qy0 = y0 / 2 - KT_CM, qx0 = x0 / 2 - KT_CM;
  for (int i = threadIdx.x; i < CH * CW; i += KT_THREADS) {
    const int cy = i / CW, cx = i - cy * CW;
    const int q = min(max(qy0 + cy, -1), p.mc), pc = min(max(qx0 + cx, -1), p.mc);
    cs[i] = __ldg(p.vc + kc_idx(p.Pc, q, pc));
  }
  for (int i = threadIdx.x; i < G::H * G::W; i += KT_THREADS) {
    const int ry = i / G::W, rx = i - ry * G::W;
    const int y = y0 - D + ry, x = x0 - D + rx;
    const size_t gi = kc_idx(P, min(max(y, -1), m), min(max(x, -1), m));
    fs[i] = __ldg(p.f + gi);
    if (!VZ) buf[1][i] = __ldg(p.u + gi);
  }
  __syncthreads();
  // stage 0: v + P vc on the full region (zero outside the interior)
  auto cp = [&](int q, int pc) { return cs[(q - qy0) * CW + (pc - qx0)]; };
  for (int i = threadIdx.x; i < G::H * G::W; i += KT_THREADS) {
    const int ry = i / G::W, rx = i - ry * G::W;
    const int y = y0 - D + ry, x = x0 - D + rx;
    double v = 0.0;
    if (y >= 0 && y < m && x >= 0 && x < m) v = DADD(VZ ? 0.0 : buf[1][i], kc_prolong_val(y, x, cp));
    buf[0][i] = v;
  }
  __syncthreads();
  int cur = 0;
#pragma unroll 1
  for (int t = 1; t <= NU; ++t) {
    const int h = D - t;
    const int rh = KT_TY + 1 + 2 * h, rw = KT_TX + 1 + 2 * h;
    const double* src = buf[cur];
    double* dst = buf[cur ^ 1];
    for (int i = threadIdx.x; i < rh * rw; i += KT_THREADS) {
      const int ry = i / rw, rx = i - ry * rw;
      const int y = y0 - h + ry, x = x0 - h + rx;
      const int k = (ry + t) * G::W + (rx + t);
      dst[k] = (y >= 0 && y < m && x >= 0 && x < m) ? kc_jacobi_pt(src[k], fs[k], kc_apply9(src + k, G::W, s), s.c)
                                                     : 0.0;
    }
    __syncthreads();
    cur ^= 1;
  }
  const double* o = buf[cur];
  for (int i = threadIdx.x; i < KT_TY * KT_TX; i += KT_THREADS) {
    const int ry = i / KT_TX, rx = i - ry * KT_TX;
    const int y = y0 + ry, x = x0 + rx;
    if (y < m && x < m) p.uo[kc_idx(P, y, x)] = o[(ry + D) * G::W + (rx + D)];
  }
}

// ---------------------------------------------------------------------------
// Column tiles (k_ctile_pre): the same pass with one lane per region column
// and each warp owning a block of RB rows, so every stage is RB independent
// chains per thread with 3 shared-memory loads per row and no index
// division.  Region W = TX + 1 + 2D <= 32 columns (TX = 24 owned at D = 3),
// H = TY + 1 + 2D rows; rows and columns outside the interior are +0.0 at
// every stage (Dirichlet), as in k_tile_pre.
// ---------------------------------------------------------------------------
#define KC_CT_TX 24
#define KC_CT_NW 8
__device__ __forceinline__ void kt_cp8(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}

template <int NU, bool ZERO, int TY, int NW = KC_CT_NW>
__global__ void __launch_bounds__(NW * 32) k_ctile_pre(const TileParams p) {
  constexpr int D = NU + 1;
  constexpr int TX = KC_CT_TX;
  constexpr int W = TX + 1 + 2 * D;
  constexpr int H = TY + 1 + 2 * D;
  constexpr int RB = (H - 2 + NW - 1) / NW;  // rows per warp (stage 1)
  static_assert(W <= 32, "one lane per region column");
  __shared__ double su[2][H][32];
  __shared__ double sf[H][32];
  // a programmatically launched successor (the bottom kernel) may start its
  // independent prologue on free SMs now; it waits for this grid itself
  asm volatile("griddepcontrol.launch_dependents;");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tx = blockIdx.x % p.tiles_x, ty = blockIdx.x / p.tiles_x;
  const int y0 = ty * TY, x0 = tx * TX;
  const int m = p.m, P = p.P;
  const St9 s = p.s;
  const int gx = x0 - D + lane;  // global column of this lane
  const bool xin = gx >= 0 && gx < m;
  // load f (and u) of the region: lane = column, rows strided over warps;
  // coordinates outside [-1, m] read the all-zero ghost ring
  {
    const int cx = min(max(gx, -1), m);
    for (int r = w; r < H; r += NW) {
      const int cy = min(max(y0 - D + r, -1), m);
      if (lane < W) {
        const size_t gi = kc_idx(P, cy, cx);
        kt_cp8(&sf[r][lane], p.f + gi);
        if (!ZERO) kt_cp8(&su[0][r][lane], p.u + gi);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
#pragma unroll
  for (int t = 1; t <= D; ++t) {
    const double(*src)[32] = su[(t - 1) & 1];
    double(*dst)[32] = su[t & 1];
    const bool lane_on = lane >= t && lane < W - t;
    const int r0 = t + w * RB, r1 = min(r0 + RB, H - t);
    if (lane_on && r0 < r1) {
      double out[RB];
      if (ZERO && t == 1) {
#pragma unroll
        for (int k = 0; k < RB; ++k)
          if (r0 + k < r1) out[k] = NU > 0 ? kc_jacobi_zero(sf[r0 + k][lane], s.c) : sf[r0 + k][lane];
      } else if (r1 - r0 == RB) {  // full block: every load first, RB independent chains
        double v[RB + 2][3], fv[RB];
#pragma unroll
        for (int k = 0; k < RB + 2; ++k)
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) v[k][dx] = src[r0 - 1 + k][lane - 1 + dx];
#pragma unroll
        for (int k = 0; k < RB; ++k) fv[k] = sf[r0 + k][lane];
#pragma unroll
        for (int k = 0; k < RB; ++k) {
          const double au = kc_sum9(s, v[k][0], v[k][1], v[k][2], v[k + 1][0], v[k + 1][1], v[k + 1][2], v[k + 2][0],
                                    v[k + 2][1], v[k + 2][2]);
          out[k] = t <= NU ? kc_jacobi_pt(v[k + 1][1], fv[k], au, s.c) : DSUB(fv[k], au);
        }
      } else {
#pragma unroll
        for (int k = 0; k < RB; ++k)
          if (r0 + k < r1) {
            const int r = r0 + k;
            const double au = kc_sum9(s, src[r - 1][lane - 1], src[r - 1][lane], src[r - 1][lane + 1], src[r][lane - 1],
                                      src[r][lane], src[r][lane + 1], src[r + 1][lane - 1], src[r + 1][lane],
                                      src[r + 1][lane + 1]);
            out[k] = t <= NU ? kc_jacobi_pt(src[r][lane], sf[r][lane], au, s.c) : DSUB(sf[r][lane], au);
          }
      }
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const int r = r0 + k;
        if (r < r1) {
          const int gy = y0 - D + r;
          const double v = (xin && gy >= 0 && gy < m) ? out[k] : 0.0;
          dst[r][lane] = v;
          // v after NU sweeps: owned points straight to HBM
          if (t == NU && r >= D && r < D + TY && lane >= D && lane < D + TX && xin && gy >= 0 && gy < m)
            p.uo[kc_idx(P, gy, gx)] = v;
        }
      }
    }
    __syncthreads();
  }
  // full weighting of the residual rows y0 .. y0+TY, columns x0 .. x0+TX
  const double(*r)[32] = su[D & 1];
  for (int i = threadIdx.x; i < (TY / 2) * (TX / 2); i += NW * 32) {
    const int qy = i / (TX / 2), qx = i - qy * (TX / 2);
    const int q = y0 / 2 + qy, pc = x0 / 2 + qx;
    if (q < p.mc && pc < p.mc) {
      const int cy = D + 2 * qy + 1, cx = D + 2 * qx + 1;
      p.fc[kc_idx(p.Pc, q, pc)] = kc_fw(r[cy - 1][cx - 1], r[cy - 1][cx], r[cy - 1][cx + 1], r[cy][cx - 1], r[cy][cx],
                                        r[cy][cx + 1], r[cy + 1][cx - 1], r[cy + 1][cx], r[cy + 1][cx + 1]);
    }
  }
}

// v + P vc, then NU sweeps, on column tiles (region W = TX + 2 NU <= 32
// columns, H = TY + 2 NU rows; the coarse patch under it in shared memory)
template <int NU, bool VZ, int TY, int NW = KC_CT_NW>
__global__ void __launch_bounds__(NW * 32) k_ctile_post(const TileParams p) {
  constexpr int D = NU;
  constexpr int TX = KC_CT_TX;
  constexpr int W = TX + 2 * D;
  constexpr int H = TY + 2 * D;
  constexpr int RB = (H - 2 > 0 ? H - 2 + NW - 1 : NW) / NW;  // rows per warp in a sweep
  constexpr int R0 = (H + NW - 1) / NW;                       // rows per warp in the prolongation
  constexpr int CH = TY / 2 + D + 3;                          // coarse patch rows
  static_assert(W <= 32, "one lane per region column");
  __shared__ double su[2][H][32];
  __shared__ double sf[H][32];
  __shared__ double sc[CH][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tx = blockIdx.x % p.tiles_x, ty = blockIdx.x / p.tiles_x;
  const int y0 = ty * TY, x0 = tx * TX;
  const int m = p.m, P = p.P;
  const St9 s = p.s;
  const int gx = x0 - D + lane;
  const bool xin = gx >= 0 && gx < m;
  const int qy0 = ((y0 - D) >> 1) - 1, qx0 = ((x0 - D) >> 1) - 1;  // coarse patch origin
  {
    const int cx = min(max(gx, -1), m);
    for (int r = w; r < H; r += NW) {
      const int cy = min(max(y0 - D + r, -1), m);
      if (lane < W) {
        const size_t gi = kc_idx(P, cy, cx);
        kt_cp8(&sf[r][lane], p.f + gi);
        if (!VZ) kt_cp8(&su[1][r][lane], p.u + gi);
      }
    }
    // f and v of this level are final already (ex_ctile_post); the coarse v
    // is the previous grid's output
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int qx = min(max(qx0 + lane, -1), p.mc);
    for (int r = w; r < CH; r += NW) {
      const int qy = min(max(qy0 + r, -1), p.mc);
      kt_cp8(&sc[r][lane], p.vc + kc_idx(p.Pc, qy, qx));
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  // stage 0: v + P vc on the region (transfer.py:50-58, cycle.py:174-176)
  if (lane < W) {
    auto cp = [&](int q, int pc) { return sc[q - qy0][pc - qx0]; };
#pragma unroll
    for (int k = 0; k < R0; ++k) {
      const int r = w * R0 + k;
      if (r < H) {
        const int gy = y0 - D + r;
        double v = 0.0;
        if (xin && gy >= 0 && gy < m) v = DADD(VZ ? 0.0 : su[1][r][lane], kc_prolong_val(gy, gx, cp));
        su[0][r][lane] = v;
        if (NU == 0 && r >= D && r < D + TY && lane >= D && lane < D + TX && xin && gy >= 0 && gy < m)
          p.uo[kc_idx(P, gy, gx)] = v;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int t = 1; t <= NU; ++t) {
    const double(*src)[32] = su[(t - 1) & 1];
    double(*dst)[32] = su[t & 1];
    const bool lane_on = lane >= t && lane < W - t;
    const int r0 = t + w * RB, r1 = min(r0 + RB, H - t);
    if (lane_on && r0 < r1) {
      double out[RB];
      if (r1 - r0 == RB) {
        double v[RB + 2][3], fv[RB];
#pragma unroll
        for (int k = 0; k < RB + 2; ++k)
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) v[k][dx] = src[r0 - 1 + k][lane - 1 + dx];
#pragma unroll
        for (int k = 0; k < RB; ++k) fv[k] = sf[r0 + k][lane];
#pragma unroll
        for (int k = 0; k < RB; ++k) {
          const double au = kc_sum9(s, v[k][0], v[k][1], v[k][2], v[k + 1][0], v[k + 1][1], v[k + 1][2], v[k + 2][0],
                                    v[k + 2][1], v[k + 2][2]);
          out[k] = kc_jacobi_pt(v[k + 1][1], fv[k], au, s.c);
        }
      } else {
#pragma unroll
        for (int k = 0; k < RB; ++k)
          if (r0 + k < r1) {
            const int r = r0 + k;
            const double au = kc_sum9(s, src[r - 1][lane - 1], src[r - 1][lane], src[r - 1][lane + 1], src[r][lane - 1],
                                      src[r][lane], src[r][lane + 1], src[r + 1][lane - 1], src[r + 1][lane],
                                      src[r + 1][lane + 1]);
            out[k] = kc_jacobi_pt(src[r][lane], sf[r][lane], au, s.c);
          }
      }
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const int r = r0 + k;
        if (r < r1) {
          const int gy = y0 - D + r;
          const bool in = xin && gy >= 0 && gy < m;
          const double v = in ? out[k] : 0.0;
          if (t < NU) dst[r][lane] = v;
          else if (in && r >= D && r < D + TY && lane >= D && lane < D + TX) p.uo[kc_idx(P, gy, gx)] = v;
        }
      }
    }
    if (t < NU) __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Fused sibling passes (k_ctile_postpre): a routine call's post pass (v + P vc,
// NU2 sweeps; cycle.py:219-220) immediately followed by the NEXT call's pre
// pass on the same level (NU1 sweeps, residual, full weighting; cycle.py:211-
// 213) -- the kappa-cycle's second recursive call (cycle.py:215-218) starts
// exactly where the first one ended, so the intermediate v (after the post
// sweeps) is consumed only by the following sweeps and never leaves the
// tile.  One launch and one pass over the level instead of two, with the
// same per-point arithmetic (kc_common.cuh).  Column tiles as k_ctile_pre
// with D = NU2 + NU1 + 1 stages after the prolongation stage (region W =
// TX + 1 + 2 D <= 32 columns, so TX = 20 at D = 5).
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int kc_pp_tx(int D) { return ((32 - 1 - 2 * D) / 2) * 2; }

template <int NU2, int NU1, bool VZ, int TY, int NW = KC_CT_NW>
__global__ void __launch_bounds__(NW * 32) k_ctile_postpre(const TileParams p) {
  constexpr int NS = NU2 + NU1;  // sweeps
  constexpr int D = NS + 1;      // + the residual stage
  constexpr int TX = kc_pp_tx(D);
  constexpr int W = TX + 1 + 2 * D;
  constexpr int H = TY + 1 + 2 * D;
  constexpr int RB = (H - 2 + NW - 1) / NW;  // rows per warp in a stage
  constexpr int R0 = (H + NW - 1) / NW;      // rows per warp in the prolongation
  constexpr int CH = (H + 1) / 2 + 3;        // coarse patch rows
  static_assert(W <= 32 && TX >= 2, "one lane per region column");
  __shared__ double su[2][H][32];
  __shared__ double sf[H][32];
  __shared__ double sc[CH][32];
  // a programmatically launched successor (the bottom kernel) may start its
  // independent prologue on free SMs now; it waits for this grid itself
  asm volatile("griddepcontrol.launch_dependents;");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tx = blockIdx.x % p.tiles_x, ty = blockIdx.x / p.tiles_x;
  const int y0 = ty * TY, x0 = tx * TX;
  const int m = p.m, P = p.P;
  const St9 s = p.s;
  const int gx = x0 - D + lane;
  const bool xin = gx >= 0 && gx < m;
  const int qy0 = ((y0 - D) >> 1) - 1, qx0 = ((x0 - D) >> 1) - 1;  // coarse patch origin
  {
    const int cx = min(max(gx, -1), m);
    for (int r = w; r < H; r += NW) {
      const int cy = min(max(y0 - D + r, -1), m);
      if (lane < W) {
        const size_t gi = kc_idx(P, cy, cx);
        kt_cp8(&sf[r][lane], p.f + gi);
        if (!VZ) kt_cp8(&su[1][r][lane], p.u + gi);
      }
    }
    // this level's f and v are final already; the coarse v is the previous
    // grid's output (and the coarse f, written below, its input)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int qx = min(max(qx0 + lane, -1), p.mc);
    for (int r = w; r < CH; r += NW) {
      const int qy = min(max(qy0 + r, -1), p.mc);
      kt_cp8(&sc[r][lane], p.vc + kc_idx(p.Pc, qy, qx));
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  // stage 0: v + P vc on the region (transfer.py:50-58, cycle.py:174-176)
  if (lane < W) {
    auto cp = [&](int q, int pc) { return sc[q - qy0][pc - qx0]; };
#pragma unroll
    for (int k = 0; k < R0; ++k) {
      const int r = w * R0 + k;
      if (r < H) {
        const int gy = y0 - D + r;
        double v = 0.0;
        if (xin && gy >= 0 && gy < m) v = DADD(VZ ? 0.0 : su[1][r][lane], kc_prolong_val(gy, gx, cp));
        su[0][r][lane] = v;
        if (NS == 0 && r >= D && r < D + TY && lane >= D && lane < D + TX && xin && gy >= 0 && gy < m)
          p.uo[kc_idx(P, gy, gx)] = v;
      }
    }
  }
  __syncthreads();
  // stages 1 .. NS: the NU2 post sweeps then the NU1 pre sweeps; stage D:
  // the residual f - A v
#pragma unroll
  for (int t = 1; t <= D; ++t) {
    const double(*src)[32] = su[(t - 1) & 1];
    double(*dst)[32] = su[t & 1];
    const bool lane_on = lane >= t && lane < W - t;
    const int r0 = t + w * RB, r1 = min(r0 + RB, H - t);
    if (lane_on && r0 < r1) {
      double out[RB];
      if (r1 - r0 == RB) {  // full block: every load first, RB independent chains
        double v[RB + 2][3], fv[RB];
#pragma unroll
        for (int k = 0; k < RB + 2; ++k)
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) v[k][dx] = src[r0 - 1 + k][lane - 1 + dx];
#pragma unroll
        for (int k = 0; k < RB; ++k) fv[k] = sf[r0 + k][lane];
#pragma unroll
        for (int k = 0; k < RB; ++k) {
          const double au = kc_sum9(s, v[k][0], v[k][1], v[k][2], v[k + 1][0], v[k + 1][1], v[k + 1][2], v[k + 2][0],
                                    v[k + 2][1], v[k + 2][2]);
          out[k] = t <= NS ? kc_jacobi_pt(v[k + 1][1], fv[k], au, s.c) : DSUB(fv[k], au);
        }
      } else {
#pragma unroll
        for (int k = 0; k < RB; ++k)
          if (r0 + k < r1) {
            const int r = r0 + k;
            const double au = kc_sum9(s, src[r - 1][lane - 1], src[r - 1][lane], src[r - 1][lane + 1], src[r][lane - 1],
                                      src[r][lane], src[r][lane + 1], src[r + 1][lane - 1], src[r + 1][lane],
                                      src[r + 1][lane + 1]);
            out[k] = t <= NS ? kc_jacobi_pt(src[r][lane], sf[r][lane], au, s.c) : DSUB(sf[r][lane], au);
          }
      }
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const int r = r0 + k;
        if (r < r1) {
          const int gy = y0 - D + r;
          const double v = (xin && gy >= 0 && gy < m) ? out[k] : 0.0;
          dst[r][lane] = v;
          // v after all NS sweeps: owned points straight to HBM
          if (t == NS && r >= D && r < D + TY && lane >= D && lane < D + TX && xin && gy >= 0 && gy < m)
            p.uo[kc_idx(P, gy, gx)] = v;
        }
      }
    }
    __syncthreads();
  }
  // full weighting of the residual rows y0 .. y0+TY, columns x0 .. x0+TX
  const double(*r)[32] = su[D & 1];
  for (int i = threadIdx.x; i < (TY / 2) * (TX / 2); i += NW * 32) {
    const int qy = i / (TX / 2), qx = i - qy * (TX / 2);
    const int q = y0 / 2 + qy, pc = x0 / 2 + qx;
    if (q < p.mc && pc < p.mc) {
      const int cy = D + 2 * qy + 1, cx = D + 2 * qx + 1;
      p.fc[kc_idx(p.Pc, q, pc)] = kc_fw(r[cy - 1][cx - 1], r[cy - 1][cx], r[cy - 1][cx + 1], r[cy][cx - 1], r[cy][cx],
                                        r[cy][cx + 1], r[cy + 1][cx - 1], r[cy + 1][cx], r[cy + 1][cx + 1]);
    }
  }
}
