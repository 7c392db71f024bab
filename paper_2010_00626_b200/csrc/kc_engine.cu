// kc_engine.cu — host engine and C-ABI (include/kcb200.h) of the B200-native
// kappa-cycle multigrid engine.
//
// The engine owns the per-level device storage of one solve (GridState,
// cycle.py:144-179), executes the state-protocol operations one at a time
// (the drop-in path driven by the reference's own kappa_cycle), and runs the
// native cycle: the kappa recursion (cycle.py:204-220) is flattened on the
// host into a schedule of fused HBM kernels for the fine levels and one
// persistent bottom kernel per entry into the smem-resident coarse levels,
// captured once as a CUDA graph per (kappa, level-1 buffer state).
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/kcb200.h"
#include "kc_bottom.cuh"
#include "kc_common.cuh"
#include "kc_loop.cuh"
#include "kc_grid_kernels.cuh"
#include "kc_pcg.cuh"
#include "kc_zebra.cuh"
#include "kc_stream.cuh"
#include "kc_tile.cuh"
#include "kc_strip.cuh"
#include "kc_dist.cuh"

namespace {

thread_local std::string g_create_err;

// k_stop_check inside the conditional WHILE graph of the stand-alone solve:
// it runs after the level-0 pre kernel has produced the norms of the
// current iterate v_it (cycle.py:338-353) and decides whether the rest of
// the cycle and the next iteration run (kc_loop.cuh; the loop body folds
// the same test into the norm reduction's last block)
__global__ void k_stop_check(cudaGraphConditionalHandle h_loop, cudaGraphConditionalHandle h_rest, int set_rest,
                             SolveState* st, const double* __restrict__ scal) {
  if (threadIdx.x != 0) return;
  kc_stop_test(LoopCheck{h_loop, h_rest, set_rest, st}, scal[0], scal[1]);
}

struct Level {
  int m = 0, P = 0;  // m: columns (nx); rows ny == m except under y-semi-coarsening
  int ny = 0;
  // zebra (kc_zebra.cuh): dgtsv plans of the x- and y-line systems, the
  // cross-line stencils (line row / column zeroed; the y one transposed)
  ZPlan zp[2]{};
  ZPart zpart[2]{};  // the FMA build's partition-method plans (s = 0: none)
  ZPart zpline[2]{};  // ... with KZL_K segments, one block per line (few lines, the coarsest line)
  void* zmem[2] = {nullptr, nullptr};
  void* zpmem[2] = {nullptr, nullptr};
  void* zplmem[2] = {nullptr, nullptr};
  bool zsing[2] = {false, false};
  St9 zoff[2]{};
  size_t elems = 0;
  double* v[2] = {nullptr, nullptr};
  double* f = nullptr;
  int cur = 0;
  bool vzero = false;
  St9 st{};
};

enum OpKind : int { OP_RELAX, OP_RESTRICT, OP_ZERO, OP_PROLONG, OP_COARSEST, OP_BOTTOM, OP_PRE, OP_POST, OP_POSTPRE };
#define KC_FUSE_MAXNU 4      // fused streaming kernels exist for nu <= 4
#define KC_FUSE_MIN_M 127    // HBM levels handled by the fused kernels
#ifndef KC_TILE_MAX_M
#define KC_TILE_MAX_M 511    // up to this side the overlapped-tile pre kernel beats streaming
#endif
#ifndef KC_TILE_POST_MAX_M
#define KC_TILE_POST_MAX_M 255  // the lag-1 streaming post pass wins from 511 up (measured 10.3 vs 12.2 us)
#endif
struct Op {
  int kind, level, a, b;
};

struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  int end_cur0 = 0;
  int kernels = 0;
};

// the whole stand-alone loop in one graph:
//   pre (level 0, input norms) ; k_stop_check ; WHILE(go) { rest of the cycle ; pre ; k_stop_check }
struct SolveGraph {
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr, pre = nullptr, rest = nullptr;
  int end_cur0 = 0, kernels_pre = 0, kernels_rest = 0;
};

}  // namespace

struct kc_handle {
  int n = 0, coarsening = 0, smoother = 0, nu1 = 0, nu2 = 0, device = 0;
  double omega = 0.0;
  std::vector<Level> L;
  int Lb = -1;  // 0-based first smem-resident (bottom) level, or -1 if none
  BotParams bot_base{};
  size_t bot_smem = 0;
  int bot_m0 = 0;
  int bot_cs = 1;  // CTAs per bottom launch (thread-block cluster when > 1)
  double* mv_mats = nullptr;  // side-15 frame operators (FMA build, kc_bottom.cuh)
  int mv_resident = 0;        // blocks resident in the bottom kernel's shared memory
  int mv_avail = 0;           // blocks computed (frames with non-resident blocks read them from L2)
  double line_w[3] = {0, 0, 0};  // semi-y coarsest line: lower, diag, upper (raw w[1][:])
  bool line_singular = false;
  // host-built bottom phase schedules, keyed by (kappa1, kappa2, v_zero)
  std::map<std::tuple<int, int, int>, std::tuple<unsigned*, int, int, int>> bot_sched;  // dev, n, final cur, mv_used
  cudaStream_t stream = nullptr;      // the stream every operation is issued on
  cudaStream_t own_stream = nullptr;  // created by kc_create (kc_set_stream may redirect `stream`)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double* d_part = nullptr;     // reduction partials
  double* d_scal = nullptr;     // device scalars
  double* h_scal = nullptr;     // pinned host mirror
  std::map<std::tuple<int, int, int, int>, GraphEntry> graphs;  // (kappa, cur0, vzero0, norms)
  std::map<std::pair<int, int>, SolveGraph> solve_graphs;       // (kappa, cur0)
  std::map<std::tuple<int, int, int>, SolveGraph> pcg_graphs;   // (kappa, measure x, cur0)
  PcgState* d_pcg = nullptr;
  double* d_pcgpart = nullptr;  // per-block partials of k_pcg_apply_dot
  double* d_npart = nullptr;  // norm partials of the fused level-1 kernels (per warp: post; per lane: pre)
  double* d_nblk = nullptr;    // block sums of k_norms_lanes
  unsigned* d_ncount = nullptr;
  int npart_cap = 0;
  bool fuse = true;           // use the fused streaming kernels in native cycles
  bool tile = true;           // overlapped-tile kernels on the mid-size levels
  bool pdl = true;            // programmatic dependent launch around the bottom kernel (KC_PDL=0: off)
  bool postpre = true;        // fused sibling post+pre passes on the column-tile levels (KC_POSTPRE=0: off)
  int zebra_few = 256;        // KZ_FEW: most lines per half-sweep for the one-line-per-block kernel
  int ctile_small_m = 255;    // column-tile pre passes with half-height tiles up to this side (KC_CTILE_SMALL_M)
  // streaming warps per SM where chunks would be short (KC_KS_SHORT_WPS): a
  // cap of 16 (round 1) now costs time -- the level-2 post pass 32 -> 29 us
  // with every resident warp (n=12 kappa=3 cycle 0.818 -> 0.813 ms)
  int ks_short_wps = 64;
  int ctile_post_small_m = 255;  // ... post passes (KC_CTILE_POST_SMALL_M)
  // the streaming k_postpre on 1023^2 and up (KC_POSTPRE_STREAM=1: on): bit-exact,
  // but as slow as the two passes it replaces (2047^2: 57 vs 32 + 27 us;
  // these passes are issue-bound, not traffic-bound), so off by default
  bool postpre_stream = false;
  int ks_sym_max = 2;         // shared products on symmetric levels: 0 off, 1 w1/w7 only, 2 all (KC_SYM)
  int num_sms = 148;
  SolveState* d_solve = nullptr;   // device loop state
  LoopCheck loop_ck{};             // while capturing the loop body: the norm reduction runs the stop test
  bool loop_ck_on = false;
  double* d_hist = nullptr;        // err | res histories for the device loop
  int hist_cap = 0;
  std::map<const void*, int> ks_occ;  // warp slots per streaming kernel (one wave)
  int launches = 0;             // kernel launches issued by the executor (for capture counting)
  std::string err;
  // PCG vectors (lazily allocated), finest padded layout
  double *x = nullptr, *p = nullptr, *ap = nullptr, *fb = nullptr;
  double* p2 = nullptr;  // the device PCG loop alternates p between p and p2
  double* snap = nullptr;  // kc_snapshot copy of the finest v
};

#define KC_FAIL(h, code, ...)                     \
  do {                                            \
    char _b[512];                                 \
    snprintf(_b, sizeof(_b), __VA_ARGS__);        \
    if (h) (h)->err = _b; else g_create_err = _b; \
    return (code);                                \
  } while (0)

#define KC_CUDA(h, call)                                                                    \
  do {                                                                                      \
    cudaError_t _e = (call);                                                                \
    if (_e != cudaSuccess) KC_FAIL(h, KC_ECUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
  } while (0)

#define KC_LAUNCH_CHECK(h) KC_CUDA(h, cudaGetLastError())

namespace {

// ---------------------------------------------------------------------------
// host Galerkin coarsening (stencil.py:126-148), exact numpy arithmetic order
// ---------------------------------------------------------------------------
struct HGrid {
  int ny, nx;
  std::vector<double> a;
  HGrid(int ny_, int nx_) : ny(ny_), nx(nx_), a((size_t)ny_ * nx_, 0.0) {}
  double get(int y, int x) const { return (y < 0 || x < 0 || y >= ny || x >= nx) ? 0.0 : a[(size_t)y * nx + x]; }
  double& at(int y, int x) { return a[(size_t)y * nx + x]; }
};

// scipy.ndimage.correlate(mode="constant", cval=0): C-order taps, taps with
// |w| <= DBL_EPSILON skipped.
HGrid h_apply(const double* w, const HGrid& u) {
  HGrid o(u.ny, u.nx);
  for (int y = 0; y < u.ny; ++y)
    for (int x = 0; x < u.nx; ++x) {
      double acc = 0.0;
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const double ww = w[(dy + 1) * 3 + (dx + 1)];
          if (std::fabs(ww) <= DBL_EPSILON) continue;
          acc = acc + ww * u.get(y + dy, x + dx);
        }
      o.at(y, x) = acc;
    }
  return o;
}

HGrid h_prolong(const HGrid& c, int coarsening) {
  if (coarsening == KC_COARSEN_FULL) {
    HGrid f(2 * c.ny + 1, 2 * c.nx + 1);
    for (int y = 0; y < f.ny; ++y)
      for (int x = 0; x < f.nx; ++x) {
        const int q = y >> 1, p = x >> 1;
        double e;
        if (y & 1) e = (x & 1) ? c.get(q, p) : 0.5 * (c.get(q, p - 1) + c.get(q, p));
        else if (x & 1) e = 0.5 * (c.get(q - 1, p) + c.get(q, p));
        else e = 0.25 * (((c.get(q - 1, p - 1) + c.get(q - 1, p)) + c.get(q, p - 1)) + c.get(q, p));
        f.at(y, x) = e;
      }
    return f;
  }
  HGrid f(2 * c.ny + 1, c.nx);  // semi-y (transfer.py:59-66)
  for (int y = 0; y < f.ny; ++y)
    for (int x = 0; x < f.nx; ++x) {
      const int q = y >> 1;
      f.at(y, x) = (y & 1) ? c.get(q, x) : 0.5 * (c.get(q - 1, x) + c.get(q, x));
    }
  return f;
}

HGrid h_restrict(const HGrid& f, int coarsening) {
  if (coarsening == KC_COARSEN_FULL) {
    HGrid c((f.ny - 1) / 2, (f.nx - 1) / 2);
    for (int q = 0; q < c.ny; ++q)
      for (int p = 0; p < c.nx; ++p) {
        const int y = 2 * q + 1, x = 2 * p + 1;
        const double edge = ((f.get(y - 1, x) + f.get(y + 1, x)) + f.get(y, x - 1)) + f.get(y, x + 1);
        const double corner =
            ((f.get(y - 1, x - 1) + f.get(y - 1, x + 1)) + f.get(y + 1, x - 1)) + f.get(y + 1, x + 1);
        c.at(q, p) = ((4.0 * f.get(y, x) + 2.0 * edge) + corner) / 16.0;
      }
    return c;
  }
  HGrid c((f.ny - 1) / 2, f.nx);  // semi-y (transfer.py:84-86)
  for (int q = 0; q < c.ny; ++q)
    for (int x = 0; x < c.nx; ++x)
      c.at(q, x) = 0.25 * ((f.get(2 * q, x) + 2.0 * f.get(2 * q + 1, x)) + f.get(2 * q + 2, x));
  return c;
}

void h_galerkin(const double* w, int coarsening, double* out) {
  const int m = 7, cy = 3, cx = 3;  // _AUX_COARSE (stencil.py:123)
  HGrid c(m, m);
  c.at(cy, cx) = 1.0;
  HGrid resp = h_restrict(h_apply(w, h_prolong(c, coarsening)), coarsening);
  for (int dy = -1; dy <= 1; ++dy)
    for (int dx = -1; dx <= 1; ++dx) out[(dy + 1) * 3 + (dx + 1)] = resp.get(cy - dy, cx - dx);
}

dim3 grid2(int mx, int my, int ry = 1) {
  return dim3((unsigned)((mx + KC_BX - 1) / KC_BX), (unsigned)((my + KC_BY * ry - 1) / (KC_BY * ry)));
}
const dim3 kBlock(KC_BX, KC_BY);

// ---------------------------------------------------------------------------
// executor: one reference state-protocol operation -> kernels on h->stream
// ---------------------------------------------------------------------------
int ex_materialize(kc_handle* h, int l) {
  Level& L = h->L[l];
  if (!L.vzero) return KC_OK;
  k_zero<<<grid2(L.m, L.ny), kBlock, 0, h->stream>>>(L.v[L.cur], L.ny, L.m, L.P);
  KC_LAUNCH_CHECK(h);
  ++h->launches;
  L.vzero = false;
  return KC_OK;
}

// LAPACK dgtsv elimination of a constant-coefficient tridiagonal system of
// order n (what scipy.linalg.solve_banded((1,1)) runs, smoother.py:133),
// recorded as a plan: everything but the right-hand-side updates is data
// independent.  Host fp64 without contraction (-ffp-contract=off).
struct HostZPlan {
  std::vector<double> fact, d, du, dl;
  std::vector<unsigned char> piv;
  bool singular = false;
};
HostZPlan gtsv_plan(double lo, double di, double up, int n) {
  HostZPlan p;
  std::vector<double> dl(n > 1 ? n - 1 : 0, lo), d(n, di), du(n > 1 ? n - 1 : 0, up);
  p.fact.assign(n > 1 ? n - 1 : 0, 0.0);
  p.piv.assign(n > 1 ? n - 1 : 0, 0);
  for (int i = 0; i < n - 1; ++i) {
    if (std::fabs(d[i]) >= std::fabs(dl[i])) {
      if (d[i] == 0.0) p.singular = true;
      const double fact = dl[i] / d[i];
      p.fact[i] = fact;
      d[i + 1] = d[i + 1] - fact * du[i];
      if (i < n - 2) dl[i] = 0.0;
    } else {
      const double fact = d[i] / dl[i];
      p.fact[i] = fact;
      p.piv[i] = 1;
      d[i] = dl[i];
      const double temp = d[i + 1];
      d[i + 1] = du[i] - fact * temp;
      if (i < n - 2) {
        dl[i] = du[i + 1];
        du[i + 1] = -fact * dl[i];
      }
      du[i] = temp;
    }
  }
  if (d[n - 1] == 0.0) p.singular = true;
  p.d = d;
  p.du = du;
  p.dl.assign(dl.begin(), dl.begin() + (n > 2 ? n - 2 : 0));
  return p;
}

// Partition-method plan (kc_zebra.cuh k_zebra_solve_part) of the constant
// line system tridiag(a, d, c) of order n = K (s + 1) - 1 (FMA build).
int zpart_setup(kc_handle* h, double a, double d, double c, int n, ZPart* out, void** mem, int K = KZP_K) {
  *out = ZPart{};
  if (n < 2 * K - 1 || (n + 1) % K != 0) return KC_OK;  // short lines keep dgtsv
  const int s = (n + 1) / K - 1;
  std::vector<double> seg(4 * (size_t)s), red(2 * (size_t)(K - 1));
  double *cp = seg.data(), *m = cp + s, *p = m + s, *q = p + s;
  for (int i = 0; i < s; ++i) {
    const double den = i == 0 ? d : d - a * cp[i - 1];
    if (den == 0.0) return KC_OK;
    m[i] = 1.0 / den;
    cp[i] = c * m[i];
  }
  auto thomas = [&](std::vector<double> b, double* x) {  // T_s x = b with the factors above
    std::vector<double> z(s);
    for (int i = 0; i < s; ++i) z[i] = (b[i] - (i ? a * z[i - 1] : 0.0)) * m[i];
    x[s - 1] = z[s - 1];
    for (int i = s - 2; i >= 0; --i) x[i] = z[i] - cp[i] * x[i + 1];
  };
  std::vector<double> e0(s, 0.0), e1(s, 0.0);
  e0[0] = a;
  e1[s - 1] = c;
  thomas(e0, p);
  thomas(e1, q);
  const double ra = -a * p[s - 1], rd = d - a * q[s - 1] - c * p[0], rc = -c * q[0];
  double *rcp = red.data(), *rm = rcp + (K - 1);
  for (int j = 0; j < K - 1; ++j) {
    const double den = j == 0 ? rd : rd - ra * rcp[j - 1];
    if (den == 0.0) return KC_OK;
    rm[j] = 1.0 / den;
    rcp[j] = rc * rm[j];
  }
  const size_t bytes = sizeof(double) * (seg.size() + red.size());
  KC_CUDA(h, cudaMalloc(mem, bytes));
  double* dv = reinterpret_cast<double*>(*mem);
  KC_CUDA(h, cudaMemcpy(dv, seg.data(), sizeof(double) * seg.size(), cudaMemcpyHostToDevice));
  KC_CUDA(h, cudaMemcpy(dv + seg.size(), red.data(), sizeof(double) * red.size(), cudaMemcpyHostToDevice));
  *out = ZPart{dv, dv + seg.size(), a, c, ra, s};
  return KC_OK;
}

int zebra_setup(kc_handle* h, const double* w) {
  for (int l = 0; l < h->n; ++l) {
    Level& L = h->L[l];
    const double* wl = w + 9 * l;  // raw (un-dropped) coefficients build the line systems
    for (int axis = 0; axis < 2; ++axis) {
      const bool need = (axis == 0 && (h->smoother == KC_SMOOTH_ZEBRA_X || h->smoother == KC_SMOOTH_ZEBRA_XY)) ||
                        (axis == 1 && (h->smoother == KC_SMOOTH_ZEBRA_Y || h->smoother == KC_SMOOTH_ZEBRA_XY));
      if (!need) continue;
      const int n = axis == 0 ? L.m : L.ny;
      const HostZPlan hp = axis == 0 ? gtsv_plan(wl[3], wl[4], wl[5], n) : gtsv_plan(wl[1], wl[4], wl[7], n);
      L.zsing[axis] = hp.singular;
#if KC_FAST
      {  // the partition-method plan (dgtsv never pivots on these dominant systems)
        bool pivots = false;
        for (unsigned char pv : hp.piv) pivots |= pv != 0;
        if (!pivots && !hp.singular) {
          const int rc = axis == 0 ? zpart_setup(h, wl[3], wl[4], wl[5], n, &L.zpart[axis], &L.zpmem[axis])
                                   : zpart_setup(h, wl[1], wl[4], wl[7], n, &L.zpart[axis], &L.zpmem[axis]);
          if (rc) return rc;
          const int rc2 = axis == 0
                              ? zpart_setup(h, wl[3], wl[4], wl[5], n, &L.zpline[axis], &L.zplmem[axis], KZL_K)
                              : zpart_setup(h, wl[1], wl[4], wl[7], n, &L.zpline[axis], &L.zplmem[axis], KZL_K);
          if (rc2) return rc2;
        }
      }
#endif
      std::vector<double> rd(hp.d.size());
      for (size_t i = 0; i < rd.size(); ++i) rd[i] = 1.0 / hp.d[i];  // the FMA build's back substitution
      const size_t nd = hp.fact.size() + hp.d.size() + hp.du.size() + hp.dl.size() + rd.size();
      const size_t bytes = sizeof(double) * (nd + 1) + hp.piv.size() + 16;
      KC_CUDA(h, cudaMalloc(&L.zmem[axis], bytes));
      std::vector<char> host(bytes, 0);
      double* hd = reinterpret_cast<double*>(host.data());
      size_t o = 0;
      auto put = [&](const std::vector<double>& v) {
        const size_t at = o;
        for (double x : v) hd[o++] = x;
        return at;
      };
      const size_t of = put(hp.fact), od = put(hp.d), odu = put(hp.du), odl = put(hp.dl), ord = put(rd);
      unsigned char* hpv = reinterpret_cast<unsigned char*>(hd + nd + 1);
      for (size_t i = 0; i < hp.piv.size(); ++i) hpv[i] = hp.piv[i];
      KC_CUDA(h, cudaMemcpy(L.zmem[axis], host.data(), bytes, cudaMemcpyHostToDevice));
      const double* dd = reinterpret_cast<const double*>(L.zmem[axis]);
      L.zp[axis] = ZPlan{dd + of, dd + od, dd + odu, dd + odl,
                         reinterpret_cast<const unsigned char*>(dd + nd + 1), n, dd + ord};
      // cross-line stencil: the line's row (x-lines) or column (y-lines) of
      // taps zeroed; y-lines accumulate in the transposed C order
      St9 off{};
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) off.w[a * 3 + b] = axis == 0 ? L.st.w[a * 3 + b] : L.st.w[b * 3 + a];
      off.w[3] = off.w[4] = off.w[5] = 0.0;
      L.zoff[axis] = off;
    }
  }
  if (h->coarsening == KC_COARSEN_SEMI_Y) {  // Thomas pivots of the coarsest line (smoother.py:77-85)
    const double* wl = w + 9 * (h->n - 1);
    h->line_w[0] = wl[3];
    h->line_w[1] = wl[4];
    h->line_w[2] = wl[5];
    double piv = wl[4];
    bool sing = piv == 0.0;
    double cp = sing ? 0.0 : wl[5] / piv;
    for (int i = 1; i < h->L[h->n - 1].m && !sing; ++i) {
      piv = wl[4] - wl[3] * cp;
      if (piv == 0.0) sing = true;
      else cp = wl[5] / piv;
    }
    h->line_singular = sing;
  }
  return KC_OK;
}

// few long lines per half-sweep (y-semi-coarsened levels): the FMA build
// solves one line per block with KZL_K segments (n = 12 zebra-x + semi-y
// kappa=2: 35.3 -> 30.4 ms per cycle with the threshold 256; the aspect
// condition keeps full coarsening on the 32-segment kernel, which the
// one-line kernel slows down there: 9.05 -> 9.65 ms)
#define KZ_FEW(nl, len) ((nl) <= h->zebra_few && (len) >= 4 * (nl))
// One zebra sweep with lines along x (axis 0) or y (axis 1), in place:
// even lines, then odd lines with the updated even ones (smoother.py:107-135)
int ex_zebra(kc_handle* h, int l, int axis) {
  Level& L = h->L[l];
  if (L.zsing[axis]) KC_FAIL(h, KC_ESINGULAR, "singular tridiagonal line system");
  int rc = ex_materialize(h, l);
  if (rc) return rc;
  double* u = L.v[L.cur];
  for (int par = 0; par < 2; ++par) {
    if (axis == 0) {
      if (par >= L.ny) break;
      const int nl = (L.ny - par + 1) / 2;
      k_zebra_rhs_x<<<dim3((L.m + 31) / 32, (nl + 7) / 8), dim3(32, 8), 0, h->stream>>>(u, L.f, L.ny, L.m, L.P,
                                                                                       L.zoff[0], par);
      if (L.zpline[0].s && KZ_FEW(nl, L.m)) {
        k_zebra_solve_line<true><<<nl, KZL_K, sizeof(double) * 4 * L.zpline[0].s, h->stream>>>(u, u, L.P, L.zpline[0],
                                                                                             par);
      } else if (L.zpart[0].s) {
        const size_t sm = sizeof(double) * (4 * (size_t)L.zpart[0].s + (size_t)KZP_K * 32 * (KZP_TC + 1));
        KC_CUDA(h, cudaFuncSetAttribute(k_zebra_solve_part_x, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k_zebra_solve_part_x<<<(nl + 31) / 32, KZP_K * 32, sm, h->stream>>>(u, L.P, L.zpart[0], par, nl);
      }
      else
        k_zebra_solve_x<<<(nl + 63) / 64, 64, 0, h->stream>>>(u, L.ny, L.P, L.zp[0], par);
    } else {
      if (par >= L.m) break;
      const int nl = (L.m - par + 1) / 2;
      k_zebra_rhs_y<<<dim3((nl + 31) / 32, (L.ny + 7) / 8), dim3(32, 8), 0, h->stream>>>(u, L.f, L.ny, L.m, L.P,
                                                                                        L.zoff[1], par);
      if (L.zpline[1].s && KZ_FEW(nl, L.ny))
        k_zebra_solve_line<false><<<nl, KZL_K, sizeof(double) * 4 * L.zpline[1].s, h->stream>>>(u, u, L.P,
                                                                                              L.zpline[1], par);
      else if (L.zpart[1].s)
        k_zebra_solve_part<false><<<(nl + 31) / 32, KZP_K * 32, sizeof(double) * 4 * L.zpart[1].s, h->stream>>>(
            u, L.P, L.zpart[1], par, nl);
      else
        k_zebra_solve_y<<<(nl + 63) / 64, 64, 0, h->stream>>>(u, L.m, L.P, L.zp[1], par);
    }
    KC_LAUNCH_CHECK(h);
    h->launches += 2;
  }
  return KC_OK;
}

int ex_zebra(kc_handle* h, int l, int axis);
int ex_relax(kc_handle* h, int l, int count) {
  Level& L = h->L[l];
  if (h->smoother != KC_SMOOTH_JACOBI) {  // relax(), smoother.py:138-163
    if (h->smoother == KC_SMOOTH_ZEBRA_XY && count % 2)
      KC_FAIL(h, KC_EINVAL, "alternating zebra needs an even relaxation count");
    const int reps = h->smoother == KC_SMOOTH_ZEBRA_XY ? count / 2 : count;
    for (int it = 0; it < reps; ++it) {
      int rc;
      if (h->smoother != KC_SMOOTH_ZEBRA_Y && (rc = ex_zebra(h, l, 0))) return rc;
      if (h->smoother != KC_SMOOTH_ZEBRA_X && (rc = ex_zebra(h, l, 1))) return rc;
    }
    return KC_OK;
  }
  for (int it = 0; it < count; ++it) {
    double* u = L.v[L.cur];
    double* o = L.v[L.cur ^ 1];
    if (L.vzero) k_jacobi<true><<<grid2(L.m, L.ny, KC_RY), kBlock, 0, h->stream>>>(u, L.f, o, L.ny, L.m, L.P, L.st);
    else k_jacobi<false><<<grid2(L.m, L.ny, KC_RY), kBlock, 0, h->stream>>>(u, L.f, o, L.ny, L.m, L.P, L.st);
    KC_LAUNCH_CHECK(h);
    ++h->launches;
    L.vzero = false;
    L.cur ^= 1;
  }
  return KC_OK;
}

int ex_restrict(kc_handle* h, int l) {
  Level& L = h->L[l];
  Level& C = h->L[l + 1];
  if (h->coarsening == KC_COARSEN_SEMI_Y) {  // transfer.py:84-86
    if (L.vzero)
      k_resid_restrict_semi<true><<<grid2(C.m, C.ny), kBlock, 0, h->stream>>>(L.v[L.cur], L.f, C.f, C.ny, C.m, L.P,
                                                                            C.P, L.st);
    else
      k_resid_restrict_semi<false><<<grid2(C.m, C.ny), kBlock, 0, h->stream>>>(L.v[L.cur], L.f, C.f, C.ny, C.m, L.P,
                                                                             C.P, L.st);
  } else if (L.vzero) {
    k_resid_restrict<true><<<grid2(C.m, C.ny), kBlock, 0, h->stream>>>(L.v[L.cur], L.f, C.f, C.ny, C.m, L.P, C.P,
                                                                     L.st);
  } else {
    k_resid_restrict<false><<<grid2(C.m, C.ny), kBlock, 0, h->stream>>>(L.v[L.cur], L.f, C.f, C.ny, C.m, L.P, C.P,
                                                                      L.st);
  }
  KC_LAUNCH_CHECK(h);
  ++h->launches;
  return KC_OK;
}

int ex_prolong(kc_handle* h, int l) {
  Level& L = h->L[l];
  Level& C = h->L[l + 1];
  int rc = ex_materialize(h, l + 1);
  if (rc) return rc;
  if (h->coarsening == KC_COARSEN_SEMI_Y) {  // transfer.py:59-66
    if (L.vzero)
      k_prolong_add_semi<true><<<grid2(L.m, L.ny), kBlock, 0, h->stream>>>(L.v[L.cur], C.v[C.cur], L.ny, L.m, L.P, C.P);
    else
      k_prolong_add_semi<false><<<grid2(L.m, L.ny), kBlock, 0, h->stream>>>(L.v[L.cur], C.v[C.cur], L.ny, L.m, L.P,
                                                                          C.P);
  } else if (L.vzero) {
    k_prolong_add<true><<<grid2(L.m, L.ny), kBlock, 0, h->stream>>>(L.v[L.cur], C.v[C.cur], L.ny, L.m, L.P, C.P);
  } else {
    k_prolong_add<false><<<grid2(L.m, L.ny), kBlock, 0, h->stream>>>(L.v[L.cur], C.v[C.cur], L.ny, L.m, L.P, C.P);
  }
  KC_LAUNCH_CHECK(h);
  ++h->launches;
  L.vzero = false;
  return KC_OK;
}

int ex_coarsest(kc_handle* h) {
  Level& L = h->L[h->n - 1];
  if (L.ny == 1 && L.m > 1 && h->coarsening == KC_COARSEN_SEMI_Y) {  // one x-line, cycle.py:191-200
    if (h->line_singular) KC_FAIL(h, KC_ESINGULAR, "zero pivot in tridiagonal elimination");
    if (L.zpline[0].s)  // FMA build: the partition method on the single line (its own x-line system)
      k_zebra_solve_line<true><<<1, KZL_K, sizeof(double) * 4 * L.zpline[0].s, h->stream>>>(L.v[L.cur], L.f, L.P,
                                                                                           L.zpline[0], 0);
    else
      k_coarsest_line<<<1, 32, 0, h->stream>>>(L.v[L.cur], L.f, L.v[L.cur ^ 1], L.m, L.P, h->line_w[0],
                                               h->line_w[1], h->line_w[2]);
    KC_LAUNCH_CHECK(h);
    ++h->launches;
    L.vzero = false;
    return KC_OK;
  }
  if (L.m != 1 || L.ny != 1) KC_FAIL(h, KC_EINVAL, "not a coarsest grid: shape (%d, %d)", L.ny, L.m);
  if (L.st.center == 0.0) KC_FAIL(h, KC_ESINGULAR, "singular coarsest operator");
  k_coarsest<<<1, 32, 0, h->stream>>>(L.v[L.cur], L.f, L.P, L.st.center);
  KC_LAUNCH_CHECK(h);
  ++h->launches;
  L.vzero = false;
  return KC_OK;
}

int get_bot_sched(kc_handle* h, int k1, int k2, int vzero, const unsigned** dev, int* n, int* final_cur,
                  int* mv_used) {
  auto key = std::make_tuple(k1, k2, vzero);
  auto it = h->bot_sched.find(key);
  if (it == h->bot_sched.end()) {
    BotBuilder b;
    b.m0 = h->bot_m0;
    b.nlev = h->bot_base.nlev;
    b.nu1 = h->nu1;
    b.nu2 = h->nu2;
    b.vz = vzero ? 1u : 0u;
    b.nstrip = h->bot_base.nstrip;
    b.mv_mask = (unsigned)h->mv_avail;
    b.deep = h->bot_base.deep;
    b.deep0 = h->bot_base.deep0 != 0;
    if (b.nlev > 1) b.top(k1, k2);
    if ((int)b.out.size() > KC_BOT_MAXPH)
      KC_FAIL(h, KC_EINVAL, "bottom schedule of %zu phases exceeds %d", b.out.size(), KC_BOT_MAXPH);
    unsigned* d = nullptr;
    const size_t bytes = sizeof(unsigned) * (b.out.empty() ? 1 : b.out.size());
    KC_CUDA(h, cudaMalloc(&d, bytes));
    if (!b.out.empty()) KC_CUDA(h, cudaMemcpy(d, b.out.data(), sizeof(unsigned) * b.out.size(), cudaMemcpyHostToDevice));
    it = h->bot_sched.emplace(key, std::make_tuple(d, (int)b.out.size(), (int)(b.cur & 1u), (int)b.mv_used)).first;
  }
  *dev = std::get<0>(it->second);
  *n = std::get<1>(it->second);
  *final_cur = std::get<2>(it->second);
  *mv_used = std::get<3>(it->second);
  return KC_OK;
}

// k_bottom's dynamic shared-memory limit is a per-function attribute shared
// by every handle of this library: only ever raise it (a smaller handle
// created later must not break the launches or graphs of a larger one).
cudaError_t bot_smem_attr(size_t bytes) {
  static size_t cur = 0;
  if (bytes <= cur) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k_bottom, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

// Side-15 frame operators of the FMA build (kc_bottom.cuh "Frame operators"):
// columns computed on the device by k_tiny_mats, then as many blocks made
// resident in every CTA of the cluster as its shared memory holds, in the
// order the kappa-cycles use them (B1, B2, A1, B3, A2, A3).  Frames whose
// blocks are not resident keep the interpreter path.
int setup_frame_operators(kc_handle* h, const cudaDeviceProp& prop) {
  BotParams& bp = h->bot_base;
  int d15 = -1;
  for (int d = 0; d < bp.nlev; ++d)
    if (bot_m(h->bot_m0, d) == KC_MV_M) d15 = d;
  if (d15 < bp.nstrip || d15 + 4 != bp.nlev) return KC_OK;
  BotParams tp{};
  tp.deep = -1;
  tp.nlev = 4;
  tp.nu1 = h->nu1;
  tp.nu2 = h->nu2;
  for (int j = 0; j < 4; ++j) tp.st[j] = bp.st[d15 + j];
  bot_geometry(tp, KC_MV_M, 1);
  const size_t mbytes = sizeof(double) * KC_MV_NBLK * (size_t)KC_MV_N * KC_MV_LD;
  KC_CUDA(h, cudaMalloc(&h->mv_mats, mbytes));
  KC_CUDA(h, cudaMemset(h->mv_mats, 0, mbytes));
  // with the pair operators (KC_TINY_PAIRS=0: the side-31 calls keep two frames)
  const char* penv = getenv("KC_TINY_PAIRS");
  const bool pairs = !(penv && penv[0] == '0');
  k_tiny_mats<<<dim3(2 * KC_MV_N, pairs ? 6 : 3), 256, sizeof(double) * tp.total>>>(tp, h->mv_mats);
  KC_LAUNCH_CHECK(h);
  KC_CUDA(h, cudaDeviceSynchronize());
  cudaFuncAttributes fa{};
  KC_CUDA(h, cudaFuncGetAttributes(&fa, k_bottom));
  const size_t smem_max = prop.sharedMemPerBlockOptin - fa.sharedSizeBytes;
  const int R = (KC_MV_N + h->bot_cs - 1) / h->bot_cs;
  const int off = (bp.total + 1) & ~1;
  const size_t per = sizeof(double) * (size_t)R * KC_MV_LD;
  // residency: the blocks the side-31 frames use first (B1 and the pairs),
  // then the single frames' in the order the kappa-cycles use them
  const int order[KC_MV_NBLK] = {1, KC_MV_PAIR0, KC_MV_PAIR0 + 1, KC_MV_PAIR0 + 2, 3, 0, 5, 2, 4};
  int mask = 0, nres = 0;
  for (int b = 0; b < KC_MV_NBLK; ++b) bp.mv_slot[b] = -1;  // not resident: bot_mv_frame reads it from global (L2)
  for (int b : order) {
    if (b >= KC_MV_PAIR0 && !pairs) continue;
    if (sizeof(double) * (size_t)(off + 2 * KC_MV_N) + per * (size_t)(nres + 1) > smem_max) break;
    mask |= 1 << b;
    bp.mv_slot[b] = nres++;
  }
  if (!mask) return KC_OK;
  bp.mv_mats = h->mv_mats;
  bp.mv_off = off;
  bp.mv_rows = R;
  bp.mv_xin = off + nres * R * KC_MV_LD;
  const size_t bytes = sizeof(double) * (size_t)(bp.mv_xin + 2 * KC_MV_N);
  // the cluster must still fit with the larger shared memory
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(h->bot_cs);
  cfg.blockDim = dim3(KC_BOT_THREADS);
  cfg.dynamicSmemBytes = bytes;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = h->bot_cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (bot_smem_attr(bytes) != cudaSuccess || cudaOccupancyMaxActiveClusters(&ncl, k_bottom, &cfg) != cudaSuccess ||
      ncl < 1) {
    cudaGetLastError();
    return KC_OK;  // keep the interpreter frames
  }
  h->mv_resident = mask;
  h->mv_avail = pairs ? (1 << KC_MV_NBLK) - 1 : (1 << KC_MV_PAIR0) - 1;
  h->bot_smem = bytes;
  return KC_OK;
}

int ex_bottom(kc_handle* h, int l, int k1, int k2) {
  Level& L = h->L[l];
  BotParams bp = h->bot_base;
  bp.gv = L.v[L.cur];
  bp.gf = L.f;
  bp.gP = L.P;
  bp.v_zero = L.vzero ? 1 : 0;
  int rc = get_bot_sched(h, k1, k2, bp.v_zero, &bp.sched, &bp.nsched, &bp.final_cur, &bp.mv_copy);
  bp.mv_copy &= h->mv_resident;  // the prologue copies the resident blocks the schedule uses
  bp.mv_avail = h->mv_avail;     // the frames (device) use every block the schedule (host) assumed
  if (rc) return rc;
  if (h->L[h->n - 1].st.center == 0.0) KC_FAIL(h, KC_ESINGULAR, "singular coarsest operator");
  if (h->bot_cs > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(h->bot_cs);
    cfg.blockDim = dim3(KC_BOT_THREADS);
    cfg.dynamicSmemBytes = h->bot_smem;
    cfg.stream = h->stream;
    // programmatic dependent launch: the cluster takes free SMs and runs its
    // prologue while the previous pass (a column-tile pre pass, which
    // triggers at its start) finishes; k_bottom waits before its entry load
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = h->bot_cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    KC_CUDA(h, cudaLaunchKernelEx(&cfg, k_bottom, bp, h->bot_m0));
  } else {
    k_bottom<<<1, KC_BOT_THREADS, h->bot_smem, h->stream>>>(bp, h->bot_m0);
  }
  KC_LAUNCH_CHECK(h);
  ++h->launches;
  L.vzero = false;
  // coarser levels are scratch of the bottom kernel: logically overwritten
  for (int j = l + 1; j < h->n; ++j) h->L[j].vzero = true;
  return KC_OK;
}

// ---------------------------------------------------------------------------
// fused streaming kernels (kc_stream.cuh)
// ---------------------------------------------------------------------------
inline int ks_npb(int D) { return (KS_BAND - 1 - D - 2 * ((D + 2) / 2)) / 2; }  // KsGeom<D>::NPB

// One wave of warps: every band gets K = slots / nbands warps, each streaming
// a contiguous run of ceil((mc+1)/K) coarse rows, so all warps finish
// together and the per-warp warm-up stays a small fraction of its rows.
int ks_choose_nq(int mc, int nbands, int slots) {
  const int minnq = 2;
  const int k = slots / nbands > 1 ? slots / nbands : 1;
  const int nq = (mc + 1 + k - 1) / k;
  return nq > minnq ? nq : minnq;
}

typedef void (*KsFn)(StreamParams);
// sym: 1 if the level's stencil has w7 == w1 bitwise, 2 if it is moreover
// point-symmetric with w0 == -w2 (ks_step<SYM>); the shared products are
// instantiated for the nu = 2 passes that stream level 1
int ks_sym(const St9& s) {
  auto eq = [](double a, double b) { return std::memcmp(&a, &b, sizeof(double)) == 0; };
  if (!eq(s.w[1], s.w[7])) return 0;
  if (eq(s.w[0], s.w[8]) && eq(s.w[2], s.w[6]) && eq(s.w[3], s.w[5]) && eq(s.w[0], -s.w[2])) return 2;
  return 1;
}
KsFn ks_pre_fn(int nu, bool zero, bool norms = false, int sym = 0) {
  if (sym == 2 && nu == 2 && !zero) return norms ? k_pre<2, false, true, false, 2> : k_pre<2, false, false, false, 2>;
  if (sym && nu == 2 && !zero) return norms ? k_pre<2, false, true, false, 1> : k_pre<2, false, false, false, 1>;
#define KS_PRE(N) return zero ? k_pre<N, true> : (norms ? k_pre<N, false, true> : k_pre<N, false>)
  switch (nu) {
    case 0: KS_PRE(0);
    case 1: KS_PRE(1);
    case 2: KS_PRE(2);
    case 3: KS_PRE(3);
    case 4: KS_PRE(4);
  }
#undef KS_PRE
  return nullptr;
}
// the post pass keeps SYM = 1: with all products shared it needs 100
// registers instead of 78 (5 instead of 6 blocks per SM) and level-1 post
// slows down 94 -> 102 us, while the pre pass gains 112 -> 107 us (exact)
KsFn ks_post_fn(int nu, bool vz, int nm, int sym = 0) {
  if (sym && nu == 2 && nm == 0) return vz ? k_post<2, true, 0, false, 1> : k_post<2, false, 0, false, 1>;
#define KS_POST(N)                                                                            \
  return vz ? (nm == 1 ? k_post<N, true, 1> : nm == 2 ? k_post<N, true, (N > 0 ? 2 : 0)> : k_post<N, true, 0>) \
            : (nm == 1 ? k_post<N, false, 1> : nm == 2 ? k_post<N, false, (N > 0 ? 2 : 0)> : k_post<N, false, 0>)
  switch (nu) {
    case 0: KS_POST(0);
    case 1: KS_POST(1);
    case 2: KS_POST(2);
    case 3: KS_POST(3);
    case 4: KS_POST(4);
  }
#undef KS_POST
  return nullptr;
}

int ks_slots(kc_handle* h, const void* fn, int D) {
  auto it = h->ks_occ.find(fn);
  if (it != h->ks_occ.end()) return it->second;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ks_smem_bytes(D));
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, 128, ks_smem_bytes(D)) != cudaSuccess || blocks < 1)
    blocks = 1;
  const int slots = blocks * 4 * h->num_sms;
  h->ks_occ[fn] = slots;
  return slots;
}

StreamParams ks_params(kc_handle* h, int l, int D, int* nwarps, const void* fn) {
  Level& L = h->L[l];
  Level& C = h->L[l + 1];
  StreamParams p{};
  p.u = L.v[L.cur];
  p.f = L.f;
  p.uo = L.v[L.cur ^ 1];
  p.fc = C.f;
  p.vc = C.v[C.cur];
  p.m = L.m;
  p.P = L.P;
  p.mc = C.m;
  p.Pc = C.P;
  p.s = L.st;
  p.rows = L.m;
  p.gy0 = 0;
  p.mg = L.m;
  p.hb = 1;
  p.mcr = C.m;
  p.hbc = 1;
  p.nbands = (C.m + 1 + ks_npb(D) - 1) / ks_npb(D);
  const int slots = fn ? ks_slots(h, fn, D) : 148 * 12;
  p.nq = ks_choose_nq(C.m, p.nbands, slots);
  // where the chunks would be short (warm-up rows 2D+1 > 10 % of the streamed
  // rows), at most ks_short_wps warps per SM (default: no cap)
  if (10 * (2 * D + 1) > 2 * p.nq) p.nq = ks_choose_nq(C.m, p.nbands, std::min(slots, h->ks_short_wps * h->num_sms));
  *nwarps = p.nbands * ((C.m + 1 + p.nq - 1) / p.nq);
  return p;
}

typedef void (*KtFn)(TileParams);
KtFn kt_pre_fn(int nu, bool zero) {
#define KT_PRE(N) return zero ? k_tile_pre<N, true> : k_tile_pre<N, false>
  switch (nu) {
    case 0: KT_PRE(0);
    case 1: KT_PRE(1);
    case 2: KT_PRE(2);
    case 3: KT_PRE(3);
    case 4: KT_PRE(4);
  }
#undef KT_PRE
  return nullptr;
}
KtFn kt_post_fn(int nu, bool vz) {
#define KT_POST(N) return vz ? k_tile_post<N, true> : k_tile_post<N, false>
  switch (nu) {
    case 0: KT_POST(0);
    case 1: KT_POST(1);
    case 2: KT_POST(2);
    case 3: KT_POST(3);
    case 4: KT_POST(4);
  }
#undef KT_POST
  return nullptr;
}

int ex_tile(kc_handle* h, int l, bool pre) {
  Level& L = h->L[l];
  Level& C = h->L[l + 1];
  TileParams p{};
  p.u = L.v[L.cur];
  p.f = L.f;
  p.uo = L.v[L.cur ^ 1];
  p.fc = C.f;
  p.vc = C.v[C.cur];
  p.m = L.m;
  p.P = L.P;
  p.mc = C.m;
  p.Pc = C.P;
  p.s = L.st;
  p.tiles_x = (L.m + KT_TX - 1) / KT_TX;
  const int tiles = p.tiles_x * ((L.m + KT_TY - 1) / KT_TY);
  const int nu = pre ? h->nu1 : h->nu2;
  const int D = pre ? nu + 1 : (nu > 0 ? nu : 1);
  const size_t smem = sizeof(double) * (size_t)kt_smem_doubles(D);
  KtFn fn = pre ? kt_pre_fn(nu, L.vzero) : kt_post_fn(nu, L.vzero);
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fn<<<tiles, KT_THREADS, smem, h->stream>>>(p);
  KC_LAUNCH_CHECK(h);
  ++h->launches;
  if (!pre || nu > 0) {
    L.cur ^= 1;
    L.vzero = false;
  }
  return KC_OK;
}

// the same pre pass on column tiles (k_ctile_pre, nu1 <= 2)
#ifndef KC_CTILE_MAX_M
// column tiles measured faster than the streaming pre pass up to here; the
// FMA build's trimmed streaming pass now wins at 1023^2 (n=12 kappa=3 cycle
// 0.829 -> 0.823 ms, kappa=2 0.516 -> 0.512 ms; exact build: neutral)
#define KC_CTILE_MAX_M (KC_FAST ? 511 : 1023)
#endif
#define KC_CTILE_TY 32
int ex_ctile_pre(kc_handle* h, int l) {
  Level& L = h->L[l];
  Level& C = h->L[l + 1];
  TileParams p{};
  p.u = L.v[L.cur];
  p.f = L.f;
  p.uo = L.v[L.cur ^ 1];
  p.fc = C.f;
  p.vc = C.v[C.cur];
  p.m = L.m;
  p.P = L.P;
  p.mc = C.m;
  p.Pc = C.P;
  p.s = L.st;
  p.tiles_x = (L.m + KC_CT_TX - 1) / KC_CT_TX;
  const int nu = h->nu1;
  const bool z = L.vzero;
  // small levels: half-height tiles, so the grid covers the SMs (255^2: 88
  // tiles of 32 rows on 148 SMs; KC_CTILE_SMALL_M=0: off)
  const bool small = L.m <= h->ctile_small_m && nu == 2;
  const int ty = small ? KC_CTILE_TY / 2 : KC_CTILE_TY;
  const int tiles = p.tiles_x * ((L.m + ty - 1) / ty);
  auto fn = small ? (z ? k_ctile_pre<2, true, KC_CTILE_TY / 2> : k_ctile_pre<2, false, KC_CTILE_TY / 2>)
          : nu == 0 ? (z ? k_ctile_pre<0, true, KC_CTILE_TY> : k_ctile_pre<0, false, KC_CTILE_TY>)
          : nu == 1 ? (z ? k_ctile_pre<1, true, KC_CTILE_TY> : k_ctile_pre<1, false, KC_CTILE_TY>)
                    : (z ? k_ctile_pre<2, true, KC_CTILE_TY> : k_ctile_pre<2, false, KC_CTILE_TY>);
  fn<<<tiles, KC_CT_NW * 32, 0, h->stream>>>(p);
  KC_LAUNCH_CHECK(h);
  ++h->launches;
  if (nu > 0) {
    L.cur ^= 1;
    L.vzero = false;
  }
  return KC_OK;
}

// prolong_add + relax(nu2) on column tiles (k_ctile_post, nu2 <= 4)
#ifndef KC_CTILE_POST_MAX_M
#define KC_CTILE_POST_MAX_M 511  // faster than the streaming post pass up to here (tools/micro/midlev.cu)
#endif
#define KC_CTILE_POST_TY 16
#ifndef KC_PP_TY
#define KC_PP_TY 16  // rows per fused post+pre tile
#endif
#ifndef KC_PP_MAX_M
#define KC_PP_MAX_M 511
#endif
#ifndef KC_PP_STREAM_MIN_M
#define KC_PP_STREAM_MIN_M 1023  // streaming k_postpre on the larger levels
#endif
int ex_ctile_post(kc_handle* h, int l) {
  Level& L = h->L[l];
  Level& C = h->L[l + 1];
  TileParams p{};
  p.u = L.v[L.cur];
  p.f = L.f;
  p.uo = L.v[L.cur ^ 1];
  p.vc = C.v[C.cur];
  p.m = L.m;
  p.P = L.P;
  p.mc = C.m;
  p.Pc = C.P;
  p.s = L.st;
  p.tiles_x = (L.m + KC_CT_TX - 1) / KC_CT_TX;
  const bool z = L.vzero;
  // small levels: half-height tiles (KC_CTILE_POST_SMALL_M)
  const bool small = L.m <= h->ctile_post_small_m && h->nu2 == 2;
  const int ty = small ? KC_CTILE_POST_TY / 2 : KC_CTILE_POST_TY;
  const int tiles = p.tiles_x * ((L.m + ty - 1) / ty);
#define KCT_POST(N) (z ? k_ctile_post<N, true, KC_CTILE_POST_TY> : k_ctile_post<N, false, KC_CTILE_POST_TY>)
  void (*fn)(TileParams) = nullptr;
  if (small) fn = z ? k_ctile_post<2, true, KC_CTILE_POST_TY / 2> : k_ctile_post<2, false, KC_CTILE_POST_TY / 2>;
  else switch (h->nu2) {
    case 0: fn = KCT_POST(0); break;
    case 1: fn = KCT_POST(1); break;
    case 2: fn = KCT_POST(2); break;
    case 3: fn = KCT_POST(3); break;
    default: fn = KCT_POST(4); break;
  }
#undef KCT_POST
  // programmatic dependent launch: f and v of this level are final before
  // the previous kernel (the child's last pass or the bottom kernel, which
  // triggers only after its own wait) completes, so they are fetched before
  // k_ctile_post waits for the coarse v
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles);
  cfg.blockDim = dim3(KC_CT_NW * 32);
  cfg.stream = h->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  KC_CUDA(h, cudaLaunchKernelEx(&cfg, fn, p));
  KC_LAUNCH_CHECK(h);
  ++h->launches;
  L.cur ^= 1;
  L.vzero = false;
  return KC_OK;
}

// post pass of a call + pre pass of the next call on level l, one launch
// (k_ctile_postpre); the result of both (NU2 + NU1 sweeps) lands in the
// other buffer, the restricted residual in the child's f
int ex_postpre_stream(kc_handle* h, int l) {
  Level& L = h->L[l];
  int rc = ex_materialize(h, l + 1);
  if (rc) return rc;
  const bool z = L.vzero;
  KsFn fn = nullptr;
#define KS_PP(A, B) fn = z ? k_postpre<A, B, true> : k_postpre<A, B, false>
  switch (h->nu2 * 3 + h->nu1) {
    case 0: KS_PP(0, 0); break;
    case 1: KS_PP(0, 1); break;
    case 2: KS_PP(0, 2); break;
    case 3: KS_PP(1, 0); break;
    case 4: KS_PP(1, 1); break;
    case 5: KS_PP(1, 2); break;
    case 6: KS_PP(2, 0); break;
    case 7: KS_PP(2, 1); break;
    default: KS_PP(2, 2); break;
  }
#undef KS_PP
  const int D = h->nu1 + h->nu2 + 1;
  int nw = 0;
  StreamParams p = ks_params(h, l, D, &nw, (const void*)fn);
  fn<<<(nw + 3) / 4, 128, ks_smem_bytes(D), h->stream>>>(p);  // ks_params set the smem attribute
  KC_LAUNCH_CHECK(h);
  ++h->launches;
  L.cur ^= 1;
  L.vzero = false;
  return KC_OK;
}

int ex_postpre(kc_handle* h, int l) {
  Level& L = h->L[l];
  Level& C = h->L[l + 1];
  if (L.m > KC_PP_MAX_M) return ex_postpre_stream(h, l);
  TileParams p{};
  p.u = L.v[L.cur];
  p.f = L.f;
  p.uo = L.v[L.cur ^ 1];
  p.fc = C.f;
  p.vc = C.v[C.cur];
  p.m = L.m;
  p.P = L.P;
  p.mc = C.m;
  p.Pc = C.P;
  p.s = L.st;
  const bool z = L.vzero;
  void (*fn)(TileParams) = nullptr;
  int tx = 0;
#define KCT_PP(A, B)                                                                                       \
  do {                                                                                                     \
    fn = z ? k_ctile_postpre<A, B, true, KC_PP_TY> : k_ctile_postpre<A, B, false, KC_PP_TY>;             \
    tx = kc_pp_tx(A + B + 1);                                                                              \
  } while (0)
  switch (h->nu2 * 3 + h->nu1) {
    case 0: KCT_PP(0, 0); break;
    case 1: KCT_PP(0, 1); break;
    case 2: KCT_PP(0, 2); break;
    case 3: KCT_PP(1, 0); break;
    case 4: KCT_PP(1, 1); break;
    case 5: KCT_PP(1, 2); break;
    case 6: KCT_PP(2, 0); break;
    case 7: KCT_PP(2, 1); break;
    default: KCT_PP(2, 2); break;
  }
#undef KCT_PP
  p.tiles_x = (L.m + tx - 1) / tx;
  const int tiles = p.tiles_x * ((L.m + KC_PP_TY - 1) / KC_PP_TY);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles);
  cfg.blockDim = dim3(KC_CT_NW * 32);
  cfg.stream = h->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  KC_CUDA(h, cudaLaunchKernelEx(&cfg, fn, p));
  KC_LAUNCH_CHECK(h);
  ++h->launches;
  L.cur ^= 1;
  L.vzero = false;
  return KC_OK;
}

// relax(nu1) + restrict_residual (cycle.py:211-213) in one pass; with norms
// also ||v||, ||f - A v|| of the input v into d_scal[0], d_scal[1]
int ex_pre(kc_handle* h, int l, bool norms = false) {
  Level& L = h->L[l];
  if (norms && L.vzero) KC_FAIL(h, KC_EINVAL, "fused input norms need a materialized level");
  if (L.m <= KC_CTILE_MAX_M && h->tile && !norms && h->nu1 <= 2) return ex_ctile_pre(h, l);
  if (L.m <= KC_TILE_MAX_M && h->tile && !norms) return ex_tile(h, l, true);
  int nw = 0;
  KsFn fn = ks_pre_fn(h->nu1, L.vzero, norms, std::min(h->ks_sym_max, ks_sym(L.st)));
  StreamParams p = ks_params(h, l, h->nu1 + 1, &nw, (const void*)fn);
  if (norms) {
    if (32 * nw > h->npart_cap) KC_FAIL(h, KC_EINVAL, "norm partial buffer too small (%d < %d)", h->npart_cap, 32 * nw);
    p.part = h->d_npart;
  }
  fn<<<(nw + 3) / 4, 128, ks_smem_bytes(h->nu1 + 1), h->stream>>>(p);
  KC_LAUNCH_CHECK(h);
  ++h->launches;
  if (norms) {
    const double2* part = reinterpret_cast<const double2*>(h->d_npart);
    double2* nblk = reinterpret_cast<double2*>(h->d_nblk);
    if (h->loop_ck_on)
      k_norms_lanes<true, true><<<KS_NB, 256, 0, h->stream>>>(part, nw * 32, nblk, h->d_ncount, h->d_scal, h->loop_ck);
    else
      k_norms_lanes<true><<<KS_NB, 256, 0, h->stream>>>(part, nw * 32, nblk, h->d_ncount, h->d_scal);
    KC_LAUNCH_CHECK(h);
    ++h->launches;
  }
  if (h->nu1 > 0) {
    L.cur ^= 1;
    L.vzero = false;
  }
  return KC_OK;
}

// prolong_add + relax(nu2) (cycle.py:219-220); nm = 1: with the norms of
// the result (||v||, ||f - A v|| into d_scal[0], d_scal[1]); nm = 2: with
// f . v into d_scal[S_RZN] (PCG rz of a preconditioning cycle, nu2 >= 1)
enum { S_RZ = 2, S_PAP = 3, S_MEAS = 4, S_RZN = 5 };
int ex_post(kc_handle* h, int l, int nm) {
  Level& L = h->L[l];
  Level& C = h->L[l + 1];
  int rc = ex_materialize(h, l + 1);
  if (rc) return rc;
  if (nm == 2 && h->nu2 < 1) KC_FAIL(h, KC_EINVAL, "fused r.z needs nu2 >= 1");
  if (L.m <= KC_CTILE_POST_MAX_M && h->tile && !nm && h->nu2 <= 4) return ex_ctile_post(h, l);
  if (L.m <= KC_TILE_POST_MAX_M && h->tile && !nm) return ex_tile(h, l, false);
  int nw = 0;
  const int D = h->nu2 + (nm == 1 ? 1 : 0);
  KsFn fn = ks_post_fn(h->nu2, L.vzero, nm, std::min(h->ks_sym_max, ks_sym(L.st)));
  StreamParams p = ks_params(h, l, D > 0 ? D : 1, &nw, (const void*)fn);
  p.vc = C.v[C.cur];
  if (nm) {
    const int need = nm == 2 ? 32 * nw : nw;
    if (need > h->npart_cap) KC_FAIL(h, KC_EINVAL, "norm partial buffer too small (%d < %d)", h->npart_cap, need);
    p.part = h->d_npart;
  }
  fn<<<(nw + 3) / 4, 128, ks_smem_bytes(D > 0 ? D : 1), h->stream>>>(p);
  KC_LAUNCH_CHECK(h);
  ++h->launches;
  if (nm == 1) {
    k_norms_final<<<1, 256, 0, h->stream>>>(h->d_npart, nw, h->d_scal);
    KC_LAUNCH_CHECK(h);
    ++h->launches;
  } else if (nm == 2) {
    k_norms_lanes<false><<<KS_NB, 256, 0, h->stream>>>(reinterpret_cast<const double2*>(h->d_npart), nw * 32,
                                                        reinterpret_cast<double2*>(h->d_nblk), h->d_ncount,
                                                        h->d_scal + S_RZN);
    KC_LAUNCH_CHECK(h);
    ++h->launches;
  }
  L.cur ^= 1;
  L.vzero = false;
  return KC_OK;
}

int ex_op(kc_handle* h, const Op& op) {
  switch (op.kind) {
    case OP_PRE: return ex_pre(h, op.level, op.b != 0);
    case OP_POST: return ex_post(h, op.level, op.b);
    case OP_POSTPRE: return ex_postpre(h, op.level);
    case OP_RELAX: return ex_relax(h, op.level, op.a);
    case OP_RESTRICT: return ex_restrict(h, op.level);
    case OP_ZERO: h->L[op.level].vzero = true; return KC_OK;
    case OP_PROLONG: return ex_prolong(h, op.level);
    case OP_COARSEST: return ex_coarsest(h);
    case OP_BOTTOM: return ex_bottom(h, op.level, op.a, op.b);
  }
  return KC_EINVAL;
}

bool fusable(const kc_handle* h, int l) {
  return h->fuse && h->smoother == KC_SMOOTH_JACOBI && h->coarsening == KC_COARSEN_FULL && h->nu1 <= KC_FUSE_MAXNU &&
         h->nu2 <= KC_FUSE_MAXNU && l < h->n - 1 && h->L[l].m >= KC_FUSE_MIN_M;
}

// Flatten kappa_cycle(level, kappa) (cycle.py:204-220) into ops.  `norms`
// asks the level-0 post-smoothing of this call to also produce ||v|| and
// ||f - A v|| (the stand-alone stopping test) inside the cycle.
// norms: 0 none, 1 after the cycle (fused into the level-0 post), 2 of the
// cycle's input (fused into the level-0 pre; the device solve loop), 3 the
// PCG r . z of a preconditioning cycle (fused into the level-0 post).
// the fused sibling pass (k_ctile_postpre) applies on the column-tile levels
// up to KC_PP_MAX_M: per launch (in-graph estimates from eager timings at
// n = 12, FMA build) 255^2 7.4 vs 5.6 + 5.9 us, 511^2 12.2 vs 7.7 + 7.3 us,
// but 1023^2 36 vs 12 + 14.5 us -- its 20-of-31-column tiles recompute too
// much once the level is throughput-bound
bool postpre_ok(const kc_handle* h, int l) {
  const Level& L = h->L[l];
  if (!h->postpre || h->nu1 > 2 || h->nu2 > 2) return false;
  if (L.m <= KC_PP_MAX_M) return h->tile;
  return h->postpre_stream && L.m >= KC_PP_STREAM_MIN_M;  // the streaming k_postpre above
}

void flatten(const kc_handle* h, int l, int kappa, std::vector<Op>& ops, int norms = 0) {
  const int n = h->n;
  if (l == h->Lb) {
    ops.push_back({OP_BOTTOM, l, kappa, 0});
    return;
  }
  if (l == n - 1) {
    ops.push_back({OP_COARSEST, l, 0, 0});
    return;
  }
  const bool fu = fusable(h, l);
  if (fu) {
    // the previous op is the post pass of this level's previous call (the
    // kappa-cycle's two recursive calls are adjacent): one fused pass
    if (!norms && postpre_ok(h, l) && !ops.empty() && ops.back().kind == OP_POST && ops.back().level == l &&
        ops.back().b == 0)
      ops.back() = {OP_POSTPRE, l, 0, 0};
    else
      ops.push_back({OP_PRE, l, 0, norms == 2 ? 1 : 0});
  } else {
    ops.push_back({OP_RELAX, l, h->nu1, 0});
    ops.push_back({OP_RESTRICT, l, 0, 0});
  }
  ops.push_back({OP_ZERO, l + 1, 0, 0});
  if (l + 1 == h->Lb) {
    ops.push_back({OP_BOTTOM, l + 1, kappa, kappa > 1 ? kappa - 1 : 0});
  } else {
    flatten(h, l + 1, kappa, ops);
    if (kappa > 1) {
      if (l + 1 == n - 1) {
        // redundant second coarsest solve: identical f/center, skipped (counted by CycleStats)
      } else {
        flatten(h, l + 1, kappa - 1, ops);
      }
    }
  }
  if (fu) {
    ops.push_back({OP_POST, l, 0, norms == 1 ? 1 : (norms == 3 ? 2 : 0)});
  } else {
    ops.push_back({OP_PROLONG, l, 0, 0});
    ops.push_back({OP_RELAX, l, h->nu2, 0});
  }
}

// true when flatten(norms=true) leaves ||v||, ||f-Av|| in d_scal[0..1]
bool cycle_has_norms(const kc_handle* h) { return h->Lb != 0 && fusable(h, 0); }

// norms: 0 plain, 1 with the result's norms, 3 with the PCG r . z (flatten)
int get_cycle_graph(kc_handle* h, int kappa, GraphEntry** out, int norms = 0) {
  Level& L0 = h->L[0];
  if (norms && !cycle_has_norms(h)) norms = 0;
  if (norms == 3 && h->nu2 < 1) norms = 0;
  auto key = std::make_tuple(kappa, L0.cur, L0.vzero ? 1 : 0, norms);
  auto it = h->graphs.find(key);
  if (it != h->graphs.end()) {
    *out = &it->second;
    return KC_OK;
  }
  std::vector<Op> ops;
  flatten(h, 0, kappa, ops, norms);
  // coarse levels start every cycle logically overwritten (zero_guess precedes use)
  std::vector<int> save_cur(h->n);
  std::vector<char> save_vz(h->n);
  for (int j = 0; j < h->n; ++j) {
    save_cur[j] = h->L[j].cur;
    save_vz[j] = h->L[j].vzero;
  }
  for (int j = 1; j < h->n; ++j) h->L[j].cur = 0;
  // bottom schedules live in device memory: build them before capturing
  for (const Op& op : ops)
    if (op.kind == OP_BOTTOM) {
      const unsigned* dv;
      int nn, fc, mu, rc0;
      for (int vz = 0; vz < 2; ++vz)
        if ((rc0 = get_bot_sched(h, op.a, op.b, vz, &dv, &nn, &fc, &mu))) return rc0;
    }
  GraphEntry g;
  const int l0 = h->launches;
  KC_CUDA(h, cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  int rc = KC_OK;
  for (const Op& op : ops) {
    rc = ex_op(h, op);
    if (rc) break;
  }
  cudaGraph_t graph = nullptr;
  cudaError_t ce = cudaStreamEndCapture(h->stream, &graph);
  g.kernels = h->launches - l0;
  h->launches = l0;
  g.end_cur0 = h->L[0].cur;
  for (int j = 0; j < h->n; ++j) {
    h->L[j].cur = save_cur[j];
    h->L[j].vzero = save_vz[j];
  }
  if (rc) return rc;
  if (ce != cudaSuccess) KC_FAIL(h, KC_ECUDA, "cudaStreamEndCapture: %s", cudaGetErrorString(ce));
  g.graph = graph;
  KC_CUDA(h, cudaGraphInstantiate(&g.exec, graph, 0));
  auto ins = h->graphs.emplace(key, g);
  *out = &ins.first->second;
  return KC_OK;
}

int run_cycle_graph(kc_handle* h, int kappa, int norms = 0) {
  GraphEntry* g = nullptr;
  int rc = get_cycle_graph(h, kappa, &g, norms);
  if (rc) return rc;
  KC_CUDA(h, cudaGraphLaunch(g->exec, h->stream));
  h->L[0].cur = g->end_cur0;
  h->L[0].vzero = false;
  for (int j = 1; j < h->n; ++j) {
    h->L[j].vzero = true;  // scratch after a native cycle (contents not part of the state contract)
    h->L[j].cur = 0;
  }
  return KC_OK;
}

void drop_graphs(kc_handle* h) {
  for (auto& kv : h->graphs) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
  }
  h->graphs.clear();
  for (auto& kv : h->solve_graphs) {
    SolveGraph& g = kv.second;
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
    if (g.pre) cudaGraphDestroy(g.pre);
    if (g.rest) cudaGraphDestroy(g.rest);
  }
  h->solve_graphs.clear();
  for (auto& kv : h->pcg_graphs) {
    SolveGraph& g = kv.second;
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
    if (g.pre) cudaGraphDestroy(g.pre);
    if (g.rest) cudaGraphDestroy(g.rest);
  }
  h->pcg_graphs.clear();
}

int capture_ops(kc_handle* h, const std::vector<Op>& ops, size_t i0, size_t i1, cudaGraph_t* out, int* kernels) {
  const int l0 = h->launches;
  KC_CUDA(h, cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  int rc = KC_OK;
  for (size_t i = i0; i < i1 && rc == KC_OK; ++i) rc = ex_op(h, ops[i]);
  cudaGraph_t graph = nullptr;
  cudaError_t ce = cudaStreamEndCapture(h->stream, &graph);
  *kernels = h->launches - l0;
  h->launches = l0;
  if (rc != KC_OK || ce != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    if (rc) return rc;
    KC_FAIL(h, KC_ECUDA, "cudaStreamEndCapture: %s", cudaGetErrorString(ce));
  }
  *out = graph;
  return KC_OK;
}

// Build (once per kappa and finest buffer) the stand-alone loop graph.  The
// norms of iterate v_k come out of the level-0 pre kernel of cycle k+1
// (its first stencil stage computes f - A v_k anyway); when the stop test
// fires the remainder of that cycle is skipped and v_k, still in its buffer
// (the pre kernel writes the other one), is the result.
int get_solve_graph(kc_handle* h, int kappa, SolveGraph** out) {
  Level& L0 = h->L[0];
  const auto key = std::make_pair(kappa, L0.cur);
  auto it = h->solve_graphs.find(key);
  if (it != h->solve_graphs.end()) {
    *out = &it->second;
    return KC_OK;
  }
  std::vector<Op> ops;
  flatten(h, 0, kappa, ops, 2);
  if (ops.empty() || ops[0].kind != OP_PRE || ops[0].b != 1) KC_FAIL(h, KC_EINVAL, "no fused level-0 pre kernel");
  for (const Op& op : ops)
    if (op.kind == OP_BOTTOM) {
      const unsigned* dv;
      int nn, fc, mu, rc0;
      for (int vz = 0; vz < 2; ++vz)
        if ((rc0 = get_bot_sched(h, op.a, op.b, vz, &dv, &nn, &fc, &mu))) return rc0;
    }
  std::vector<int> save_cur(h->n);
  std::vector<char> save_vz(h->n);
  for (int j = 0; j < h->n; ++j) {
    save_cur[j] = h->L[j].cur;
    save_vz[j] = h->L[j].vzero;
  }
  for (int j = 1; j < h->n; ++j) h->L[j].cur = 0;
  SolveGraph sg;
  int rc = capture_ops(h, ops, 0, 1, &sg.pre, &sg.kernels_pre);
  std::vector<int> s1_cur(h->n);  // the state after the pre op: where the loop body starts
  std::vector<char> s1_vz(h->n);
  for (int j = 0; j < h->n; ++j) {
    s1_cur[j] = h->L[j].cur;
    s1_vz[j] = h->L[j].vzero;
  }
  if (rc == KC_OK) rc = capture_ops(h, ops, 1, ops.size(), &sg.rest, &sg.kernels_rest);
  sg.end_cur0 = L0.cur;
  for (int j = 0; j < h->n; ++j) {
    h->L[j].cur = save_cur[j];
    h->L[j].vzero = save_vz[j];
  }
  if (rc) return rc;
  if (!h->d_solve) KC_CUDA(h, cudaMalloc(&h->d_solve, sizeof(SolveState)));
  // pre ; check ; WHILE(go) { rest ; pre ; check } -- the same sequence as
  // WHILE { pre ; check ; IF(go) { rest } } without a conditional node per cycle
  cudaGraph_t cg = nullptr;
  KC_CUDA(h, cudaGraphCreate(&cg, 0));
  cudaGraphConditionalHandle h_loop;
  KC_CUDA(h, cudaGraphConditionalHandleCreate(&h_loop, cg, 1, cudaGraphCondAssignDefault));
  SolveState* st = h->d_solve;
  const double* scal = h->d_scal;
  cudaGraphConditionalHandle h_none = h_loop;
  int set_rest = 0;
  void* args[] = {&h_loop, &h_none, &set_rest, &st, &scal};
  cudaKernelNodeParams kp{};
  kp.func = (void*)k_stop_check;
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(32);
  kp.kernelParams = args;
  cudaGraphNode_t pre0, chk0, wn;
  KC_CUDA(h, cudaGraphAddChildGraphNode(&pre0, cg, nullptr, 0, sg.pre));
  KC_CUDA(h, cudaGraphAddKernelNode(&chk0, cg, &pre0, 1, &kp));
  cudaGraphNodeParams wp{};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = h_loop;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  KC_CUDA(h, cudaGraphAddNode(&wn, cg, &chk0, 1, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  const char* fenv = getenv("KC_FLATBODY");
  if (fenv && fenv[0] == '0') {  // the body as three child-graph nodes (A/B)
    cudaGraphNode_t rest_node, pre_node, chk_node;
    KC_CUDA(h, cudaGraphAddChildGraphNode(&rest_node, body, nullptr, 0, sg.rest));
    KC_CUDA(h, cudaGraphAddChildGraphNode(&pre_node, body, &rest_node, 1, sg.pre));
    KC_CUDA(h, cudaGraphAddKernelNode(&chk_node, body, &pre_node, 1, &kp));
  } else {
    // the body captured straight into the conditional node's graph: one
    // flat chain of kernel nodes (rest of the cycle, pre, check) instead of
    // child-graph nodes
    for (int j = 0; j < h->n; ++j) {
      h->L[j].cur = s1_cur[j];
      h->L[j].vzero = s1_vz[j];
    }
    const int l0 = h->launches;
    KC_CUDA(h, cudaStreamBeginCaptureToGraph(h->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    for (size_t i = 1; i < ops.size() && rc == KC_OK; ++i) rc = ex_op(h, ops[i]);
    // the pre pass's norm reduction runs the stop test in its last block
    // (KC_FUSED_CHECK=0: a separate k_stop_check kernel)
    const char* cenv = getenv("KC_FUSED_CHECK");
    const bool fused_check = !(cenv && cenv[0] == '0');
    h->loop_ck = LoopCheck{h_loop, h_none, set_rest, st};
    h->loop_ck_on = fused_check;
    // KC_LOOP_PROBE=1 (loop-overhead measurement only, tools/probe_loop.py):
    // the plain pre pass, no norms, a separate check on stale norms
    const char* lpenv = getenv("KC_LOOP_PROBE");
    const bool probe = lpenv && lpenv[0] == '1';
    if (probe) {
      Op plain = ops[0];
      plain.b = 0;
      h->loop_ck_on = false;
      if (rc == KC_OK) rc = ex_op(h, plain);
    } else if (rc == KC_OK) {
      rc = ex_op(h, ops[0]);
    }
    h->loop_ck_on = false;
    if (rc == KC_OK && (!fused_check || probe)) {
      k_stop_check<<<1, 32, 0, h->stream>>>(h_loop, h_none, set_rest, st, scal);
      if (cudaGetLastError() != cudaSuccess) rc = KC_ECUDA;
    }
    cudaGraph_t same = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(h->stream, &same);
    h->launches = l0;
    for (int j = 0; j < h->n; ++j) {
      h->L[j].cur = save_cur[j];
      h->L[j].vzero = save_vz[j];
    }
    if (rc) return rc;
    if (ce != cudaSuccess) KC_FAIL(h, KC_ECUDA, "loop body capture: %s", cudaGetErrorString(ce));
  }
  KC_CUDA(h, cudaGraphInstantiate(&sg.exec, cg, 0));
  sg.graph = cg;
  auto ins = h->solve_graphs.emplace(key, sg);
  *out = &ins.first->second;
  return KC_OK;
}

// async reductions into h->d_scal[slot]
int red_dot(kc_handle* h, const double* a, const double* b, int l, int slot, bool sq) {
  Level& L = h->L[l];
  k_red_partial<0><<<KC_RED_BLOCKS, KC_RED_THREADS, 0, h->stream>>>(a, b, L.ny, L.m, L.P, L.st, h->d_part);
  KC_LAUNCH_CHECK(h);
  if (sq) k_red_final<true><<<1, KC_RED_THREADS, 0, h->stream>>>(h->d_part, KC_RED_BLOCKS, h->d_scal + slot);
  else k_red_final<false><<<1, KC_RED_THREADS, 0, h->stream>>>(h->d_part, KC_RED_BLOCKS, h->d_scal + slot);
  KC_LAUNCH_CHECK(h);
  return KC_OK;
}

int red_resnorm(kc_handle* h, const double* u, const double* f, int l, int slot) {
  Level& L = h->L[l];
  k_red_partial<1><<<KC_RED_BLOCKS, KC_RED_THREADS, 0, h->stream>>>(u, f, L.ny, L.m, L.P, L.st, h->d_part);
  KC_LAUNCH_CHECK(h);
  k_red_final<true><<<1, KC_RED_THREADS, 0, h->stream>>>(h->d_part, KC_RED_BLOCKS, h->d_scal + slot);
  KC_LAUNCH_CHECK(h);
  return KC_OK;
}

int fetch_scalars(kc_handle* h, int count) {
  KC_CUDA(h, cudaMemcpyAsync(h->h_scal, h->d_scal, sizeof(double) * count, cudaMemcpyDeviceToHost, h->stream));
  KC_CUDA(h, cudaStreamSynchronize(h->stream));
  return KC_OK;
}

int check_level(kc_handle* h, int level) {
  if (level < 1 || level > h->n) KC_FAIL(h, KC_EINVAL, "level %d out of range 1..%d", level, h->n);
  return KC_OK;
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

int kc_abi_version(void) { return KC_ABI_VERSION; }

int kc_arith_mode(void) { return KC_FAST ? KC_ARITH_FAST : KC_ARITH_EXACT; }

const char* kc_last_error(const kc_handle* h) { return h ? h->err.c_str() : g_create_err.c_str(); }

int kc_galerkin_coarsen(const double* w_fine9, int coarsening, double* w_coarse9) {
  if (!w_fine9 || !w_coarse9) KC_FAIL((kc_handle*)nullptr, KC_EINVAL, "null stencil pointer");
  if (coarsening != KC_COARSEN_FULL && coarsening != KC_COARSEN_SEMI_Y)
    KC_FAIL((kc_handle*)nullptr, KC_EINVAL, "unknown coarsening kind %d", coarsening);
  h_galerkin(w_fine9, coarsening, w_coarse9);
  return KC_OK;
}

int kc_create(int n, int coarsening, const double* w, int smoother_kind, double omega, int nu1, int nu2,
              int device, kc_handle** out) {
  kc_handle* none = nullptr;
  if (!out || !w) KC_FAIL(none, KC_EINVAL, "null argument");
  *out = nullptr;
  if (n < 1) KC_FAIL(none, KC_EINVAL, "level count must be >= 1, got %d", n);
  if (n > 15) KC_FAIL(none, KC_EINVAL, "level count %d exceeds the engine limit 15", n);
  if (coarsening != KC_COARSEN_FULL && coarsening != KC_COARSEN_SEMI_Y)
    KC_FAIL(none, KC_EINVAL, "unknown coarsening kind %d", coarsening);
  if (smoother_kind < KC_SMOOTH_JACOBI || smoother_kind > KC_SMOOTH_ZEBRA_XY)
    KC_FAIL(none, KC_EINVAL, "unknown smoother kind %d", smoother_kind);
  if (smoother_kind == KC_SMOOTH_JACOBI && !(omega > 0.0 && omega <= 1.0))
    KC_FAIL(none, KC_EINVAL, "jacobi damping must lie in (0, 1], got %g", omega);
  if (nu1 < 0 || nu2 < 0) KC_FAIL(none, KC_EINVAL, "relaxation counts must be >= 0");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    KC_FAIL(none, KC_ECUDA, "no CUDA device available (%s); the engine has no CPU fallback",
            e != cudaSuccess ? cudaGetErrorString(e) : "0 devices");
  if (device < 0 || device >= ndev) KC_FAIL(none, KC_EINVAL, "device %d out of range (%d devices)", device, ndev);
  cudaDeviceProp prop;
  KC_CUDA(none, cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) KC_FAIL(none, KC_ECUDA, "device %d is sm_%d%d; this build targets sm_100a", device, prop.major, prop.minor);
  KC_CUDA(none, cudaSetDevice(device));

  kc_handle* h = new kc_handle();
  {
    const char* penv = getenv("KC_PDL");
    h->pdl = !(penv && penv[0] == '0');
    const char* kswenv = getenv("KC_KS_SHORT_WPS");
    if (kswenv) h->ks_short_wps = std::max(1, atoi(kswenv));
    const char* csmenv = getenv("KC_CTILE_SMALL_M");
    if (csmenv) h->ctile_small_m = atoi(csmenv);
    const char* cpsenv = getenv("KC_CTILE_POST_SMALL_M");
    if (cpsenv) h->ctile_post_small_m = atoi(cpsenv);
    const char* zfenv = getenv("KC_ZEBRA_FEW");
    if (zfenv) h->zebra_few = atoi(zfenv);
    const char* ppenv = getenv("KC_POSTPRE");
    h->postpre = !(ppenv && ppenv[0] == '0');
    const char* ppsenv = getenv("KC_POSTPRE_STREAM");
    h->postpre_stream = ppsenv && ppsenv[0] == '1';
    const char* senv = getenv("KC_SYM");
    // the shared-product form only saves work when products are separately
    // rounded; in the FMA build every product is fused into its sum
    h->ks_sym_max = senv ? atoi(senv) : (KC_FAST ? 0 : 2);
  }
  h->num_sms = prop.multiProcessorCount;
  h->n = n;
  h->coarsening = coarsening;
  h->smoother = smoother_kind;
  h->omega = omega;
  h->nu1 = nu1;
  h->nu2 = nu2;
  h->device = device;
  h->L.resize(n);
  auto fail = [&](int code) {
    g_create_err = h->err;
    kc_destroy(h);
    return code;
  };
  for (int l = 0; l < n; ++l) {  // mesh.py:56-73
    Level& L = h->L[l];
    L.ny = (1 << (n - l)) - 1;
    L.m = coarsening == KC_COARSEN_SEMI_Y ? (1 << n) - 1 : L.ny;
    L.P = kc_pitch(L.m);
    L.elems = (size_t)(L.ny + 2) * L.P;
    for (int k = 0; k < 9; ++k) {
      double wk = w[9 * l + k];
      L.st.w[k] = (std::fabs(wk) <= DBL_EPSILON) ? 0.0 : wk;  // ndimage tap drop (F3)
    }
    L.st.center = w[9 * l + 4];
    if (smoother_kind == KC_SMOOTH_JACOBI && (L.m > 1 || L.ny > 1) && (nu1 + nu2) > 0 && L.st.center == 0.0) {
      h->err = "zero center coefficient";
      return fail(KC_EINVAL);
    }
    L.st.c = omega / L.st.center;  // (omega / center), smoother.py:100
    for (int b = 0; b < 3; ++b) {
      double* ptr = nullptr;
      cudaError_t ce = cudaMalloc(&ptr, L.elems * sizeof(double));
      if (ce != cudaSuccess) {
        h->err = std::string("cudaMalloc level storage: ") + cudaGetErrorString(ce);
        return fail(KC_ENOMEM);
      }
      if (cudaMemset(ptr, 0, L.elems * sizeof(double)) != cudaSuccess) {
        cudaFree(ptr);
        h->err = "cudaMemset failed";
        return fail(KC_ECUDA);
      }
      if (b < 2) L.v[b] = ptr;
      else L.f = ptr;
    }
  }
  if (cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&h->ev0) != cudaSuccess || cudaEventCreate(&h->ev1) != cudaSuccess ||
      cudaMalloc(&h->d_part, sizeof(double) * KC_RED_BLOCKS) != cudaSuccess ||
      cudaMalloc(&h->d_scal, sizeof(double) * 64) != cudaSuccess ||
      cudaMallocHost(&h->h_scal, sizeof(double) * 64) != cudaSuccess) {
    h->err = "stream/event/scratch allocation failed";
    return fail(KC_ECUDA);
  }
  h->stream = h->own_stream;
  cudaMemset(h->d_scal, 0, sizeof(double) * 64);

  // zebra line-solve plans and the semi-y coarsest line (data independent)
  if (smoother_kind != KC_SMOOTH_JACOBI || coarsening == KC_COARSEN_SEMI_Y) {
    int rc = zebra_setup(h, w);
    if (rc) return fail(rc);
  }
  // bottom (smem-resident) levels: a cluster of 16 (else 8) CTAs entering
  // at side <= 255 with the sides >= 31 in row strips, else one CTA
  // entering at side <= 63 (kc_bottom.cuh); KC_BOT_CLUSTER=0 forces one CTA.
  // Only the Jacobi / full-coarsening path has fused kernels.
  int lb = -1, cs = 1, nstrip = 0, deep = -1, deep0 = 0;
  size_t smem = 0;
  if (smoother_kind == KC_SMOOTH_JACOBI && coarsening == KC_COARSEN_FULL) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_bottom);
    const size_t smem_max = prop.sharedMemPerBlockOptin - fa.sharedSizeBytes;
    const char* env = getenv("KC_BOT_CLUSTER");
    const bool allow = !(env && env[0] == '0');
    cudaFuncSetAttribute(k_bottom, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    // largest cluster entry side: 127 measured faster than 255 (the 255^2
    // calls run as column-tile kernels on the whole GPU instead; F-cycle
    // -3 %); KC_BOT_ENTRY overrides (<= KC_CLU_MAX_M), KC_BOT_CS=8 skips 16
    const char* eenv = getenv("KC_BOT_ENTRY");
    const int clu_max = eenv ? std::min(atoi(eenv), KC_CLU_MAX_M) : KC_CLU_ENTRY_M;
    const char* csenv = getenv("KC_BOT_CS");
    const int cs_first = csenv && atoi(csenv) == 8 ? 8 : 16;
    const char* denv = getenv("KC_DEEP");
    const bool use_deep = !(denv && denv[0] == '0');
    // deep halos on the 127^2 entry strips too, zero-guess launches as one
    // PH_FRAME127 descriptor (KC_DEEP127=0: off)
    const char* d0env = getenv("KC_DEEP127");
    const bool use_deep0 = !(d0env && d0env[0] == '0');
    // smallest strip side (KC_BOT_MINSTRIP overrides): coarser levels live in CTA 0
    const char* msenv = getenv("KC_BOT_MINSTRIP");
    const int min_strip = msenv ? std::max(atoi(msenv), 31) : KC_CLU_MIN_STRIP;
    for (int csz : {16, 8}) {
      if (csz > cs_first) continue;
      if (!allow || lb >= 0) break;
      for (int e = 0; e < n && lb < 0; ++e) {
        if (h->L[e].m > clu_max) continue;
        const int m0 = h->L[e].m, nl = n - e;
        int ns = 0;
        while (ns < nl) {
          const int m = bot_m(m0, ns);
          if (m < min_strip || (m + 1) % csz != 0 || ((m + 1) / csz) % 2 != 0) break;
          ++ns;
        }
        if (ns == 0) break;  // coarser entries have no strips either
        // deep halos on the 63^2 strips (PH_FRAME63): 16 CTAs of 4 rows,
        // entry 127^2, the 31^2 level replicated below, nu = (2, 2)
        const int dp = (use_deep && csz == 16 && m0 == 127 && ns == 2 && nl == 7 && nu1 == 2 && nu2 == 2) ? 1 : -1;
        const int dp0 = (dp == 1 && use_deep0) ? 1 : 0;
        const size_t bytes = sizeof(double) * (size_t)bot_smem_doubles(m0, nl, ns, csz, dp, dp0);
        if (bytes > smem_max) continue;
        if (bot_smem_attr(bytes) != cudaSuccess) continue;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(csz);
        cfg.blockDim = dim3(KC_BOT_THREADS);
        cfg.dynamicSmemBytes = bytes;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = csz;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, k_bottom, &cfg) != cudaSuccess || ncl < 1) {
          cudaGetLastError();
          break;
        }
        lb = e;
        cs = csz;
        nstrip = ns;
        smem = bytes;
        deep = dp;
        deep0 = dp0;
      }
    }
    cudaGetLastError();
    if (lb < 0) {
      for (int l = 0; l < n; ++l)
        if (h->L[l].m <= KC_BOT_MAX_M) {
          lb = l;
          break;
        }
      if (lb >= 0) smem = sizeof(double) * (size_t)bot_smem_doubles(h->L[lb].m, n - lb);
    }
  }
  if (lb >= 0) {
    BotParams& bp = h->bot_base;
    memset(&bp, 0, sizeof(bp));
    bp.nlev = n - lb;
    bp.nu1 = nu1;
    bp.nu2 = nu2;
    bp.nstrip = nstrip;
    bp.deep = deep;
    bp.deep0 = deep0;
    // st.async frame-operator outputs / 63^2 -> 31^2 broadcast (KC_MV_ASYNC=0,
    // KC_RB_ASYNC=0: DSMEM stores + cluster barriers, the same iterates; read
    // by the jitter builds only, kc_bottom.cuh KC_ASYNC_ON)
    const char* maenv = getenv("KC_MV_ASYNC");
    const char* raenv = getenv("KC_RB_ASYNC");
    bp.async = ((maenv && maenv[0] == '0') ? 0 : 1) | ((raenv && raenv[0] == '0') ? 0 : 2);
    for (int j = 0; j < bp.nlev; ++j) bp.st[j] = h->L[lb + j].st;
    h->bot_m0 = h->L[lb].m;
    h->bot_cs = cs;
    bot_geometry(bp, h->bot_m0, cs);
    h->bot_smem = smem;
    if (bot_smem_attr(h->bot_smem) != cudaSuccess) {
      h->err = "cudaFuncSetAttribute(k_bottom) failed";
      return fail(KC_ECUDA);
    }
    h->Lb = lb;
#if KC_FAST
    const char* mvenv = getenv("KC_TINY_MV");
    if (cs > 1 && !(mvenv && mvenv[0] == '0')) {
      int rc = setup_frame_operators(h, prop);
      if (rc) return fail(rc);
    }
#endif
  }
  if (n >= 2 && h->L[0].m >= KC_FUSE_MIN_M) {  // per-warp partials of the fused level-1 norms
    int nw = 0;
    const int D = nu2 + 1;
    StreamParams p = ks_params(h, 0, D, &nw, (const void*)ks_post_fn(nu2, true, 1));
    int nw2 = 0;
    ks_params(h, 0, D, &nw2, (const void*)ks_post_fn(nu2, false, 1));
    nw = nw > nw2 ? nw : nw2;
    for (int sym = 0; sym < 2; ++sym) {
      ks_params(h, 0, nu1 + 1, &nw2, (const void*)ks_pre_fn(nu1, false, true, sym));
      nw = nw > 32 * nw2 ? nw : 32 * nw2;  // the pre kernel leaves per-lane partials
    }
    if (nu2 >= 1) {
      ks_params(h, 0, nu2, &nw2, (const void*)ks_post_fn(nu2, false, 2));
      nw = nw > 32 * nw2 ? nw : 32 * nw2;
    }
    (void)p;
    h->npart_cap = nw;
    if (cudaMalloc(&h->d_nblk, sizeof(double) * 2 * KS_NB) != cudaSuccess ||
        cudaMalloc(&h->d_ncount, sizeof(unsigned)) != cudaSuccess ||
        cudaMemset(h->d_ncount, 0, sizeof(unsigned)) != cudaSuccess ||
        cudaMalloc(&h->d_npart, sizeof(double) * 2 * (size_t)nw) != cudaSuccess) {
      h->err = "cudaMalloc norm partials failed";
      return fail(KC_ENOMEM);
    }
  }
  *out = h;
  return KC_OK;
}

int kc_destroy(kc_handle* h) {
  if (!h) return KC_OK;
  if (h->stream) cudaStreamSynchronize(h->stream);
  drop_graphs(h);
  cudaFree(h->d_solve);
  cudaFree(h->d_hist);
  cudaFree(h->d_pcg);
  cudaFree(h->d_pcgpart);
  for (Level& L : h->L) {
    cudaFree(L.v[0]);
    cudaFree(L.v[1]);
    cudaFree(L.f);
    cudaFree(L.zmem[0]);
    cudaFree(L.zmem[1]);
    cudaFree(L.zpmem[0]);
    cudaFree(L.zpmem[1]);
    cudaFree(L.zplmem[0]);
    cudaFree(L.zplmem[1]);
  }
  cudaFree(h->x);
  cudaFree(h->p);
  cudaFree(h->p2);
  cudaFree(h->ap);
  cudaFree(h->fb);
  cudaFree(h->snap);
  cudaFree(h->mv_mats);
  cudaFree(h->d_npart);
  cudaFree(h->d_nblk);
  cudaFree(h->d_ncount);
  for (auto& kv : h->bot_sched) cudaFree(std::get<0>(kv.second));
  cudaFree(h->d_part);
  cudaFree(h->d_scal);
  if (h->h_scal) cudaFreeHost(h->h_scal);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
  return KC_OK;
}

int kc_sync(kc_handle* h) {
  if (!h) return KC_EINVAL;
  KC_CUDA(h, cudaStreamSynchronize(h->stream));
  return KC_OK;
}

int kc_level_dims(kc_handle* h, int level, int* nx, int* ny) {
  if (!h) return KC_EINVAL;
  int rc = check_level(h, level);
  if (rc) return rc;
  *nx = h->L[level - 1].m;
  *ny = h->L[level - 1].ny;
  return KC_OK;
}

int kc_set(kc_handle* h, int level, int which, const double* host, long long ny, long long nx) {
  if (!h) return KC_EINVAL;
  int rc = check_level(h, level);
  if (rc) return rc;
  Level& L = h->L[level - 1];
  if (ny != L.ny || nx != L.m) KC_FAIL(h, KC_EINVAL, "shape (%lld, %lld) != level %d shape (%d, %d)", ny, nx, level, L.ny, L.m);
  double* dst = which == KC_WHICH_F ? L.f : L.v[L.cur];
  KC_CUDA(h, cudaMemcpy2DAsync(dst + kc_idx(L.P, 0, 0), sizeof(double) * L.P, host, sizeof(double) * L.m,
                               sizeof(double) * L.m, L.ny, cudaMemcpyHostToDevice, h->stream));
  KC_CUDA(h, cudaStreamSynchronize(h->stream));
  if (which != KC_WHICH_F) L.vzero = false;
  return KC_OK;
}

int kc_get(kc_handle* h, int level, int which, double* host, long long ny, long long nx) {
  if (!h) return KC_EINVAL;
  int rc = check_level(h, level);
  if (rc) return rc;
  Level& L = h->L[level - 1];
  if (ny != L.ny || nx != L.m) KC_FAIL(h, KC_EINVAL, "shape (%lld, %lld) != level %d shape (%d, %d)", ny, nx, level, L.ny, L.m);
  if (which != KC_WHICH_F) {
    rc = ex_materialize(h, level - 1);
    if (rc) return rc;
  }
  const double* src = which == KC_WHICH_F ? L.f : L.v[L.cur];
  KC_CUDA(h, cudaMemcpy2DAsync(host, sizeof(double) * L.m, src + kc_idx(L.P, 0, 0), sizeof(double) * L.P,
                               sizeof(double) * L.m, L.ny, cudaMemcpyDeviceToHost, h->stream));
  KC_CUDA(h, cudaStreamSynchronize(h->stream));
  return KC_OK;
}

int kc_relax(kc_handle* h, int level, int count) {
  if (!h) return KC_EINVAL;
  int rc = check_level(h, level);
  if (rc) return rc;
  if (count < 0) KC_FAIL(h, KC_EINVAL, "relaxation count must be >= 0, got %d", count);
  if (count > 0 && h->L[level - 1].st.center == 0.0) KC_FAIL(h, KC_EINVAL, "zero center coefficient");
  return ex_relax(h, level - 1, count);
}

int kc_restrict_residual(kc_handle* h, int level) {
  if (!h) return KC_EINVAL;
  int rc = check_level(h, level);
  if (rc) return rc;
  if (level == h->n || h->L[level - 1].ny < 3)
    KC_FAIL(h, KC_EINVAL, "fine ny must be odd and >= 3, got %d", h->L[level - 1].ny);
  return ex_restrict(h, level - 1);
}

int kc_zero_guess(kc_handle* h, int level) {
  if (!h) return KC_EINVAL;
  int rc = check_level(h, level);
  if (rc) return rc;
  h->L[level - 1].vzero = true;
  return KC_OK;
}

int kc_prolong_add(kc_handle* h, int level) {
  if (!h) return KC_EINVAL;
  int rc = check_level(h, level);
  if (rc) return rc;
  if (level == h->n) KC_FAIL(h, KC_EINVAL, "no coarser level below level %d", level);
  return ex_prolong(h, level - 1);
}

int kc_solve_coarsest(kc_handle* h) {
  if (!h) return KC_EINVAL;
  return ex_coarsest(h);
}

int kc_apply(kc_handle* h, int level, int residual, double* out, long long ny, long long nx) {
  if (!h || !out) return KC_EINVAL;
  int rc = check_level(h, level);
  if (rc) return rc;
  Level& L = h->L[level - 1];
  if (ny != L.ny || nx != L.m) KC_FAIL(h, KC_EINVAL, "shape (%lld, %lld) != level %d shape (%d, %d)", ny, nx, level, L.ny, L.m);
  if ((rc = ex_materialize(h, level - 1))) return rc;
  double* t = L.v[L.cur ^ 1];
  if (residual) k_apply<true><<<grid2(L.m, L.ny), kBlock, 0, h->stream>>>(L.v[L.cur], L.f, t, L.ny, L.m, L.P, L.st);
  else k_apply<false><<<grid2(L.m, L.ny), kBlock, 0, h->stream>>>(L.v[L.cur], L.f, t, L.ny, L.m, L.P, L.st);
  KC_LAUNCH_CHECK(h);
  KC_CUDA(h, cudaMemcpy2DAsync(out, sizeof(double) * L.m, t + kc_idx(L.P, 0, 0), sizeof(double) * L.P,
                               sizeof(double) * L.m, L.ny, cudaMemcpyDeviceToHost, h->stream));
  KC_CUDA(h, cudaStreamSynchronize(h->stream));
  return KC_OK;
}

int kc_norm2(kc_handle* h, int level, int which, double* out) {
  if (!h || !out) return KC_EINVAL;
  int rc = check_level(h, level);
  if (rc) return rc;
  Level& L = h->L[level - 1];
  if (which != KC_WHICH_F && (rc = ex_materialize(h, level - 1))) return rc;
  const double* a = which == KC_WHICH_F ? L.f : L.v[L.cur];
  if ((rc = red_dot(h, a, a, level - 1, 0, true))) return rc;
  if ((rc = fetch_scalars(h, 1))) return rc;
  *out = h->h_scal[0];
  return KC_OK;
}

int kc_residual_norm(kc_handle* h, int level, double* out) {
  if (!h || !out) return KC_EINVAL;
  int rc = check_level(h, level);
  if (rc) return rc;
  if ((rc = ex_materialize(h, level - 1))) return rc;
  Level& L = h->L[level - 1];
  if ((rc = red_resnorm(h, L.v[L.cur], L.f, level - 1, 0))) return rc;
  if ((rc = fetch_scalars(h, 1))) return rc;
  *out = h->h_scal[0];
  return KC_OK;
}

int kc_run_cycles(kc_handle* h, int kappa, int count) {
  if (!h) return KC_EINVAL;
  if (kappa < 1) KC_FAIL(h, KC_EINVAL, "cycle counter must be >= 1, got %d", kappa);
  if (kappa > h->n) kappa = h->n;  // identical to W (cycle.py:80-82; Prop 2.1)
  for (int i = 0; i < count; ++i) {
    int rc = run_cycle_graph(h, kappa);
    if (rc) return rc;
  }
  return KC_OK;
}

int kc_time_cycles(kc_handle* h, int kappa, int count, double* ms) {
  if (!h || !ms) return KC_EINVAL;
  if (kappa < 1) KC_FAIL(h, KC_EINVAL, "cycle counter must be >= 1, got %d", kappa);
  if (kappa > h->n) kappa = h->n;
  int rc;
  GraphEntry* g = nullptr;
  if ((rc = get_cycle_graph(h, kappa, &g))) return rc;  // capture outside the timed span
  KC_CUDA(h, cudaStreamSynchronize(h->stream));
  KC_CUDA(h, cudaEventRecord(h->ev0, h->stream));
  for (int i = 0; i < count; ++i)
    if ((rc = run_cycle_graph(h, kappa))) return rc;
  KC_CUDA(h, cudaEventRecord(h->ev1, h->stream));
  KC_CUDA(h, cudaEventSynchronize(h->ev1));
  float t = 0.f;
  KC_CUDA(h, cudaEventElapsedTime(&t, h->ev0, h->ev1));
  *ms = t;
  return KC_OK;
}

int kc_profile_cycle(kc_handle* h, int kappa, int max_ops, int* op_kind, int* op_level, int* op_arg,
                     double* op_ms, int* n_ops) {
  if (!h || !n_ops) return KC_EINVAL;
  if (kappa < 1) KC_FAIL(h, KC_EINVAL, "cycle counter must be >= 1, got %d", kappa);
  if (kappa > h->n) kappa = h->n;
  std::vector<Op> ops;
  flatten(h, 0, kappa, ops);
  std::vector<cudaEvent_t> ev(ops.size() + 1);
  for (auto& e : ev) KC_CUDA(h, cudaEventCreate(&e));
  for (int j = 1; j < h->n; ++j) h->L[j].cur = 0;
  int rc = KC_OK;
  KC_CUDA(h, cudaEventRecord(ev[0], h->stream));
  for (size_t i = 0; i < ops.size(); ++i) {
    if ((rc = ex_op(h, ops[i]))) break;
    KC_CUDA(h, cudaEventRecord(ev[i + 1], h->stream));
  }
  cudaError_t se = cudaStreamSynchronize(h->stream);
  int k = 0;
  if (!rc && se == cudaSuccess) {
    for (size_t i = 0; i < ops.size() && k < max_ops; ++i, ++k) {
      float t = 0.f;
      cudaEventElapsedTime(&t, ev[i], ev[i + 1]);
      if (op_kind) op_kind[k] = ops[i].kind;
      if (op_level) op_level[k] = ops[i].level + 1;
      if (op_arg) op_arg[k] = ops[i].a;
      if (op_ms) op_ms[k] = t;
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  for (int j = 1; j < h->n; ++j) {
    h->L[j].vzero = true;
    h->L[j].cur = 0;
  }
  if (rc) return rc;
  if (se != cudaSuccess) KC_FAIL(h, KC_ECUDA, "profile cycle: %s", cudaGetErrorString(se));
  *n_ops = (int)ops.size();
  return KC_OK;
}

int kc_set_option(kc_handle* h, const char* name, int value) {
  if (!h || !name) return KC_EINVAL;
  if (strcmp(name, "fuse") == 0 || strcmp(name, "tile") == 0) {
    KC_CUDA(h, cudaStreamSynchronize(h->stream));
    if (name[0] == 'f') h->fuse = value != 0;
    else h->tile = value != 0;
    drop_graphs(h);
    return KC_OK;
  }
  KC_FAIL(h, KC_EINVAL, "unknown option '%s'", name);
}

int kc_snapshot(kc_handle* h) {
  if (!h) return KC_EINVAL;
  Level& L = h->L[0];
  int rc;
  if ((rc = ex_materialize(h, 0))) return rc;
  if (!h->snap) {
    cudaError_t ce = cudaMalloc(&h->snap, L.elems * sizeof(double));
    if (ce != cudaSuccess) KC_FAIL(h, KC_ENOMEM, "cudaMalloc snapshot: %s", cudaGetErrorString(ce));
  }
  KC_CUDA(h, cudaMemcpyAsync(h->snap, L.v[L.cur], L.elems * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  return KC_OK;
}

int kc_restore(kc_handle* h) {
  if (!h) return KC_EINVAL;
  if (!h->snap) KC_FAIL(h, KC_EINVAL, "kc_restore without kc_snapshot");
  Level& L = h->L[0];
  KC_CUDA(h, cudaMemcpyAsync(L.v[L.cur], h->snap, L.elems * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  L.vzero = false;
  return KC_OK;
}

int kc_stream(kc_handle* h, void** stream) {
  if (!h || !stream) return KC_EINVAL;
  *stream = (void*)h->stream;
  return KC_OK;
}

int kc_fill_zero(kc_handle* h, int level, int which) {
  if (!h) return KC_EINVAL;
  int rc = check_level(h, level);
  if (rc) return rc;
  Level& L = h->L[level - 1];
  if (which == KC_WHICH_F) {
    k_zero<<<grid2(L.m, L.ny), kBlock, 0, h->stream>>>(L.f, L.ny, L.m, L.P);
    KC_LAUNCH_CHECK(h);
  } else {
    L.vzero = true;
    if ((rc = ex_materialize(h, level - 1))) return rc;
  }
  return KC_OK;
}

int kc_cycle_launches(kc_handle* h, int kappa, int* kernels_per_cycle) {
  if (!h || !kernels_per_cycle) return KC_EINVAL;
  if (kappa > h->n) kappa = h->n;
  GraphEntry* g = nullptr;
  int rc = get_cycle_graph(h, kappa, &g);
  if (rc) return rc;
  *kernels_per_cycle = g->kernels;
  return KC_OK;
}

int kc_solve(kc_handle* h, int kappa, int stop_mode, double target_reduction, int max_cycles, double* err_hist,
             double* res_hist, int* iterations, int* status, double* device_ms) {
  if (!h || !iterations || !status) return KC_EINVAL;
  if (kappa < 1) KC_FAIL(h, KC_EINVAL, "cycle counter must be >= 1, got %d", kappa);
  if (!(target_reduction > 1.0)) KC_FAIL(h, KC_EINVAL, "target reduction must exceed 1, got %g", target_reduction);
  if (stop_mode != KC_STOP_ERROR && stop_mode != KC_STOP_RESIDUAL) KC_FAIL(h, KC_EINVAL, "bad stop mode %d", stop_mode);
  if (kappa > h->n) kappa = h->n;
  int rc;
  if ((rc = ex_materialize(h, 0))) return rc;
  // build the graphs before timing (setup, like build_state)
  const bool fused_norms = cycle_has_norms(h);
  Level& L0 = h->L[0];
  SolveGraph* sg = nullptr;
  if (fused_norms && max_cycles > 0 && (rc = get_solve_graph(h, kappa, &sg))) return rc;
  // the device loop needs a cycle that leaves the finest buffer where it
  // found it (always true with the fused kernels: pre and post flip once each)
  const bool device_loop = sg && sg->end_cur0 == L0.cur;
  GraphEntry* g = nullptr;
  if (!device_loop && (rc = get_cycle_graph(h, kappa, &g, fused_norms))) return rc;
  if (device_loop && max_cycles + 1 > h->hist_cap) {  // setup outside the timed span
    cudaFree(h->d_hist);
    h->d_hist = nullptr;
    KC_CUDA(h, cudaMalloc(&h->d_hist, sizeof(double) * 2 * (size_t)(max_cycles + 1)));
    h->hist_cap = max_cycles + 1;
  }
  KC_CUDA(h, cudaStreamSynchronize(h->stream));
  KC_CUDA(h, cudaEventRecord(h->ev0, h->stream));
  int st = KC_STATUS_MAX_CYCLES, it = 0, streak = 0;
  if (device_loop) {
    SolveState ss{};
    ss.reduction = target_reduction;
    ss.it = 0;
    ss.max_it = max_cycles;
    ss.streak = 0;
    ss.status = KC_STATUS_MAX_CYCLES;
    ss.stop_mode = stop_mode;
    ss.err_hist = h->d_hist;
    ss.res_hist = h->d_hist + h->hist_cap;
    KC_CUDA(h, cudaMemcpyAsync(h->d_solve, &ss, sizeof(ss), cudaMemcpyHostToDevice, h->stream));
    KC_CUDA(h, cudaGraphLaunch(sg->exec, h->stream));
    KC_CUDA(h, cudaMemcpyAsync(&ss, h->d_solve, sizeof(ss), cudaMemcpyDeviceToHost, h->stream));
    KC_CUDA(h, cudaStreamSynchronize(h->stream));
    it = ss.it;
    st = ss.status;
    if (err_hist) KC_CUDA(h, cudaMemcpy(err_hist, h->d_hist, sizeof(double) * (it + 1), cudaMemcpyDeviceToHost));
    if (res_hist)
      KC_CUDA(h, cudaMemcpy(res_hist, h->d_hist + h->hist_cap, sizeof(double) * (it + 1), cudaMemcpyDeviceToHost));
    // level-state bookkeeping after it cycles (the finest buffer is unchanged)
    L0.vzero = false;
    for (int j = 1; j < h->n; ++j) {
      h->L[j].vzero = true;
      h->L[j].cur = 0;
    }
  } else {
    if ((rc = red_dot(h, L0.v[L0.cur], L0.v[L0.cur], 0, 0, true))) return rc;
    if ((rc = red_resnorm(h, L0.v[L0.cur], L0.f, 0, 1))) return rc;
    if ((rc = fetch_scalars(h, 2))) return rc;
    const double e0 = h->h_scal[0], r0 = h->h_scal[1];
    if (err_hist) err_hist[0] = e0;
    if (res_hist) res_hist[0] = r0;
    const double m0 = stop_mode == KC_STOP_ERROR ? e0 : r0;
    const double target = m0 / target_reduction;
    double cur = m0;
    if (m0 <= target) {
      st = KC_STATUS_CONVERGED;
      max_cycles = 0;
    }
    for (it = 1; it <= max_cycles; ++it) {
      if ((rc = run_cycle_graph(h, kappa, fused_norms))) return rc;
      if (!fused_norms) {
        if ((rc = red_dot(h, L0.v[L0.cur], L0.v[L0.cur], 0, 0, true))) return rc;
        if ((rc = red_resnorm(h, L0.v[L0.cur], L0.f, 0, 1))) return rc;
      }
      if ((rc = fetch_scalars(h, 2))) return rc;
      if (err_hist) err_hist[it] = h->h_scal[0];
      if (res_hist) res_hist[it] = h->h_scal[1];
      const double prev = cur;
      cur = stop_mode == KC_STOP_ERROR ? h->h_scal[0] : h->h_scal[1];
      if (cur <= target) {
        st = KC_STATUS_CONVERGED;
        break;
      }
      streak = cur > prev ? streak + 1 : 0;
      if (streak >= 5) {  // _DIVERGENCE_STREAK, cycle.py:278
        st = KC_STATUS_DIVERGED;
        break;
      }
    }
    if (it > max_cycles) it = max_cycles;
  }
  KC_CUDA(h, cudaEventRecord(h->ev1, h->stream));
  KC_CUDA(h, cudaEventSynchronize(h->ev1));
  float ms = 0.f;
  KC_CUDA(h, cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  if (device_ms) *device_ms = ms;
  *iterations = it;
  *status = st;
  return KC_OK;
}

}  // extern "C"

namespace {
int ensure_pcg_buffers(kc_handle* h) {
  const size_t bytes = h->L[0].elems * sizeof(double);
  if (!h->d_pcgpart) KC_CUDA(h, cudaMalloc(&h->d_pcgpart, sizeof(double) * (size_t)KC_PCG_BLOCKS(h->L[0].m)));
  double** bufs[5] = {&h->x, &h->p, &h->ap, &h->fb, &h->p2};
  for (double** b : bufs) {
    if (*b) continue;
    cudaError_t ce = cudaMalloc(b, bytes);
    if (ce != cudaSuccess) KC_FAIL(h, KC_ENOMEM, "cudaMalloc PCG vector: %s", cudaGetErrorString(ce));
    KC_CUDA(h, cudaMemsetAsync(*b, 0, bytes, h->stream));
  }
  return KC_OK;
}

int upload_interior(kc_handle* h, double* dst, const double* host) {
  const Level& L = h->L[0];
  KC_CUDA(h, cudaMemcpy2DAsync(dst + kc_idx(L.P, 0, 0), sizeof(double) * L.P, host, sizeof(double) * L.m,
                               sizeof(double) * L.m, L.ny, cudaMemcpyHostToDevice, h->stream));
  return KC_OK;
}

int download_interior(kc_handle* h, double* host, const double* src) {
  const Level& L = h->L[0];
  KC_CUDA(h, cudaMemcpy2DAsync(host, sizeof(double) * L.m, src + kc_idx(L.P, 0, 0), sizeof(double) * L.P,
                               sizeof(double) * L.m, L.ny, cudaMemcpyDeviceToHost, h->stream));
  return KC_OK;
}

// z = M^-1 r into L0.v[cur]; r lives in L0.f (krylov.py:81-86)
int pcg_precondition(kc_handle* h, int kappa, kc_precond_fn fn, void* ctx, std::vector<double>& hr,
                     std::vector<double>& hz) {
  Level& L0 = h->L[0];
  if (!fn) {
    L0.vzero = true;  // state.zero_guess(1); state.f[0] = r  (r is stored in f[0])
    return run_cycle_graph(h, kappa);
  }
  int rc;
  if ((rc = download_interior(h, hr.data(), L0.f))) return rc;
  KC_CUDA(h, cudaStreamSynchronize(h->stream));
  fn(hr.data(), hz.data(), L0.m, L0.m, ctx);
  if ((rc = upload_interior(h, L0.v[L0.cur], hz.data()))) return rc;
  L0.vzero = false;
  return KC_OK;
}
}  // namespace

namespace {
// The whole PCG loop of krylov.py:100-130 in one graph launch:
//   A ; k_pcg_check ; WHILE(go) { z = M r (the cycle graph, r . z fused into
//   its last kernel) ; p = z + beta p, rz = rz_next ; A ; k_pcg_check }
// with A = { Ap = A p, pAp ; x += alpha p, r -= alpha Ap, measure }.
// r lives in L0.f and z in the finest v buffer, as in the host loop.
int get_pcg_graph(kc_handle* h, int kappa, bool mx, SolveGraph** out) {
  Level& L0 = h->L[0];
  const auto key = std::make_tuple(kappa, mx ? 1 : 0, L0.cur);
  auto it = h->pcg_graphs.find(key);
  if (it != h->pcg_graphs.end()) {
    *out = &it->second;
    return KC_OK;
  }
  const int m = L0.m, P = L0.P;
  if (!h->d_pcg) KC_CUDA(h, cudaMalloc(&h->d_pcg, sizeof(PcgState)));
  // the preconditioning cycle (z = M r from a zero guess, r . z fused)
  const int cur0 = L0.cur;
  const bool vz0 = L0.vzero;
  L0.vzero = true;
  GraphEntry* g = nullptr;
  int rc = get_cycle_graph(h, kappa, &g, 3);
  L0.vzero = vz0;
  if (rc) return rc;
  if (g->end_cur0 != cur0) KC_FAIL(h, KC_EINVAL, "preconditioning cycle does not return to its buffer");
  const double* z = L0.v[cur0];
  double* r = L0.f;
  PcgState* st = h->d_pcg;
  SolveGraph sg;
  // A: Ap, pAp, x/r update, measure
  KC_CUDA(h, cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  k_pcg_apply_dot2<<<grid2((m + 1) / 2, m, KC_RY), kBlock, 0, h->stream>>>(h->p, h->ap, m, P, L0.st, h->d_pcgpart);
  k_red_final<false><<<1, KC_RED_THREADS, 0, h->stream>>>(h->d_pcgpart, KC_PCG_BLOCKS2(m), h->d_scal + S_PAP);
  if (mx)
    k_pcg_update_xr<true><<<KC_RED_BLOCKS, KC_RED_THREADS, 0, h->stream>>>(h->x, r, h->p, h->ap, m, P, h->d_scal, S_RZ,
                                                                            S_PAP, h->d_part, st);
  else
    k_pcg_update_xr<false><<<KC_RED_BLOCKS, KC_RED_THREADS, 0, h->stream>>>(h->x, r, h->p, h->ap, m, P, h->d_scal,
                                                                             S_RZ, S_PAP, h->d_part, st);
  k_red_final<true><<<1, KC_RED_THREADS, 0, h->stream>>>(h->d_part, KC_RED_BLOCKS, h->d_scal + S_MEAS);
  cudaError_t ce = cudaStreamEndCapture(h->stream, &sg.pre);
  if (ce != cudaSuccess) KC_FAIL(h, KC_ECUDA, "PCG capture: %s", cudaGetErrorString(ce));
  // tail of the body: p = z + beta p ; rz = rz_next
  KC_CUDA(h, cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  k_pcg_update_p<<<KC_RED_BLOCKS, KC_RED_THREADS, 0, h->stream>>>(h->p, z, m, P, h->d_scal, S_RZN, S_RZ);
  k_copy_scalar<<<1, 32, 0, h->stream>>>(h->d_scal, S_RZ, S_RZN);
  ce = cudaStreamEndCapture(h->stream, &sg.rest);
  if (ce != cudaSuccess) KC_FAIL(h, KC_ECUDA, "PCG capture: %s", cudaGetErrorString(ce));
  sg.kernels_pre = 4;
  sg.kernels_rest = g->kernels + 2;
  // the body's tail fused with the next A (KC_PCG_FUSED=0: separate kernels):
  // p_new = z + beta p_old and A p_new in one pass, p alternating between
  // the two buffers, so the loop body holds two iterations (the second under
  // an IF node the first check sets)
  const char* pfenv = getenv("KC_PCG_FUSED");
  const bool fused = !(pfenv && pfenv[0] == '0');
  cudaGraph_t tail_a[2] = {nullptr, nullptr};
  if (fused) {
    for (int b = 0; b < 2; ++b) {
      double* pin = b ? h->p2 : h->p;
      double* pout = b ? h->p : h->p2;
      KC_CUDA(h, cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
      k_pcg_update_p_apply_dot2<<<grid2((m + 1) / 2, m, KC_RY), kBlock, 0, h->stream>>>(
          z, pin, pout, h->ap, m, P, L0.st, h->d_scal, S_RZN, S_RZ, h->d_pcgpart);
      k_copy_scalar<<<1, 32, 0, h->stream>>>(h->d_scal, S_RZ, S_RZN);
      k_red_final<false><<<1, KC_RED_THREADS, 0, h->stream>>>(h->d_pcgpart, KC_PCG_BLOCKS2(m), h->d_scal + S_PAP);
      if (mx)
        k_pcg_update_xr<true><<<KC_RED_BLOCKS, KC_RED_THREADS, 0, h->stream>>>(h->x, r, pout, h->ap, m, P, h->d_scal,
                                                                                S_RZ, S_PAP, h->d_part, st);
      else
        k_pcg_update_xr<false><<<KC_RED_BLOCKS, KC_RED_THREADS, 0, h->stream>>>(h->x, r, pout, h->ap, m, P,
                                                                                 h->d_scal, S_RZ, S_PAP, h->d_part, st);
      k_red_final<true><<<1, KC_RED_THREADS, 0, h->stream>>>(h->d_part, KC_RED_BLOCKS, h->d_scal + S_MEAS);
      ce = cudaStreamEndCapture(h->stream, &tail_a[b]);
      if (ce != cudaSuccess) KC_FAIL(h, KC_ECUDA, "PCG capture: %s", cudaGetErrorString(ce));
    }
  }
  // A ; check ; WHILE(go) { cycle ; tail ; A ; check } -- the sequence of
  // WHILE { A ; check ; IF(go) { cycle ; tail } } without the IF node
  cudaGraph_t cg = nullptr;
  KC_CUDA(h, cudaGraphCreate(&cg, 0));
  cudaGraphConditionalHandle h_loop;
  KC_CUDA(h, cudaGraphConditionalHandleCreate(&h_loop, cg, 1, cudaGraphCondAssignDefault));
  const double* scal = h->d_scal;
  int s_rz = S_RZ, s_pap = S_PAP, s_meas = S_MEAS, set_body = 0;
  cudaGraphConditionalHandle h_body = h_loop;
  void* args[] = {&h_loop, &h_body, &set_body, &st, &scal, &s_rz, &s_pap, &s_meas};
  cudaKernelNodeParams kp{};
  kp.func = (void*)k_pcg_check;
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(32);
  kp.kernelParams = args;
  cudaGraphNode_t a0, chk0, wn;
  KC_CUDA(h, cudaGraphAddChildGraphNode(&a0, cg, nullptr, 0, sg.pre));
  KC_CUDA(h, cudaGraphAddKernelNode(&chk0, cg, &a0, 1, &kp));
  cudaGraphNodeParams wp{};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = h_loop;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  KC_CUDA(h, cudaGraphAddNode(&wn, cg, &chk0, 1, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  if (fused) {
    // WHILE { cycle ; tailA(p -> p2) ; check (also sets the IF) ;
    //         IF(go) { cycle ; tailA(p2 -> p) ; check } }
    cudaGraphConditionalHandle h_if;
    KC_CUDA(h, cudaGraphConditionalHandleCreate(&h_if, body, 0, cudaGraphCondAssignDefault));
    int set1 = 1;
    void* args1[] = {&h_loop, &h_if, &set1, &st, &scal, &s_rz, &s_pap, &s_meas};
    cudaKernelNodeParams kp1 = kp;
    kp1.kernelParams = args1;
    cudaGraphNode_t c1, t1, k1, ifn, c2, t2, k2;
    KC_CUDA(h, cudaGraphAddChildGraphNode(&c1, body, nullptr, 0, g->graph));
    KC_CUDA(h, cudaGraphAddChildGraphNode(&t1, body, &c1, 1, tail_a[0]));
    KC_CUDA(h, cudaGraphAddKernelNode(&k1, body, &t1, 1, &kp1));
    cudaGraphNodeParams ip{};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = h_if;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    KC_CUDA(h, cudaGraphAddNode(&ifn, body, &k1, 1, &ip));
    cudaGraph_t ib = ip.conditional.phGraph_out[0];
    KC_CUDA(h, cudaGraphAddChildGraphNode(&c2, ib, nullptr, 0, g->graph));
    KC_CUDA(h, cudaGraphAddChildGraphNode(&t2, ib, &c2, 1, tail_a[1]));
    KC_CUDA(h, cudaGraphAddKernelNode(&k2, ib, &t2, 1, &kp));
    KC_CUDA(h, cudaGraphInstantiate(&sg.exec, cg, 0));
    sg.graph = cg;
    sg.end_cur0 = cur0;
    auto ins = h->pcg_graphs.emplace(key, sg);
    *out = &ins.first->second;
    return KC_OK;
  }
  cudaGraphNode_t cyc_node, tail_node, a_node, chk_node;
  KC_CUDA(h, cudaGraphAddChildGraphNode(&cyc_node, body, nullptr, 0, g->graph));
  KC_CUDA(h, cudaGraphAddChildGraphNode(&tail_node, body, &cyc_node, 1, sg.rest));
  KC_CUDA(h, cudaGraphAddChildGraphNode(&a_node, body, &tail_node, 1, sg.pre));
  KC_CUDA(h, cudaGraphAddKernelNode(&chk_node, body, &a_node, 1, &kp));
  KC_CUDA(h, cudaGraphInstantiate(&sg.exec, cg, 0));
  sg.graph = cg;
  sg.end_cur0 = cur0;
  auto ins = h->pcg_graphs.emplace(key, sg);
  *out = &ins.first->second;
  return KC_OK;
}
}  // namespace

extern "C" int kc_pcg(kc_handle* h, int kappa, const double* f, const double* x0, int stop_mode,
                      double target_reduction, int max_it, kc_precond_fn precond, void* ctx, double* hist,
                      int* iterations, int* status, int* n_precond, double* x_out, double* device_ms) {
  if (!h || !f || !iterations || !status) return KC_EINVAL;
  if (kappa < 1) KC_FAIL(h, KC_EINVAL, "cycle counter must be >= 1, got %d", kappa);
  if (!(target_reduction > 1.0)) KC_FAIL(h, KC_EINVAL, "target reduction must exceed 1, got %g", target_reduction);
  if (stop_mode != KC_STOP_ERROR && stop_mode != KC_STOP_RESIDUAL) KC_FAIL(h, KC_EINVAL, "bad stop mode %d", stop_mode);
  if (kappa > h->n) kappa = h->n;
  int rc;
  if ((rc = ensure_pcg_buffers(h))) return rc;
  Level& L0 = h->L[0];
  const int m = L0.m, P = L0.P;
  std::vector<double> hr, hz;
  const bool mx = stop_mode == KC_STOP_ERROR;
  // the whole loop on the device when the preconditioner is the native cycle
  // and the fused kernels apply (r . z fused into the cycle's last kernel)
  const bool device_loop = !precond && cycle_has_norms(h) && h->nu2 >= 1 && max_it > 0;
  SolveGraph* pg = nullptr;
  if (precond) {
    hr.resize((size_t)m * m);
    hz.resize((size_t)m * m);
  } else if (device_loop) {  // setup outside the timed span
    if ((rc = get_pcg_graph(h, kappa, mx, &pg))) return rc;
    if (max_it + 1 > h->hist_cap) {
      cudaFree(h->d_hist);
      h->d_hist = nullptr;
      KC_CUDA(h, cudaMalloc(&h->d_hist, sizeof(double) * 2 * (size_t)(max_it + 1)));
      h->hist_cap = max_it + 1;
    }
  } else {
    GraphEntry* g = nullptr;  // capture both level-1 states up front (setup)
    if ((rc = get_cycle_graph(h, kappa, &g))) return rc;
  }
  if ((rc = upload_interior(h, h->fb, f))) return rc;
  if (x0) {
    if ((rc = upload_interior(h, h->x, x0))) return rc;
  } else {
    KC_CUDA(h, cudaMemsetAsync(h->x, 0, L0.elems * sizeof(double), h->stream));
  }
  KC_CUDA(h, cudaStreamSynchronize(h->stream));
  double* r = L0.f;
  int napp = 0;
  KC_CUDA(h, cudaEventRecord(h->ev0, h->stream));
  k_pcg_residual<<<KC_RED_BLOCKS, KC_RED_THREADS, 0, h->stream>>>(h->x, h->fb, r, m, P, L0.st);
  KC_LAUNCH_CHECK(h);
  if ((rc = red_dot(h, mx ? h->x : r, mx ? h->x : r, 0, S_MEAS, true))) return rc;
  if ((rc = fetch_scalars(h, S_MEAS + 1))) return rc;
  const double norm0 = h->h_scal[S_MEAS];
  const double target = norm0 / target_reduction;
  if (hist) hist[0] = norm0;
  int st = KC_STATUS_MAX_CYCLES, it = 0;
  double cur = norm0;
  if (norm0 <= target) {
    st = KC_STATUS_CONVERGED;
  } else if (device_loop) {
    L0.vzero = true;  // z = M r from the zero guess, r . z into S_RZN
    if ((rc = run_cycle_graph(h, kappa, 3))) return rc;
    KC_CUDA(h, cudaMemcpyAsync(h->p, L0.v[L0.cur], L0.elems * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
    k_copy_scalar<<<1, 32, 0, h->stream>>>(h->d_scal, S_RZ, S_RZN);
    KC_LAUNCH_CHECK(h);
    PcgState ps{};
    ps.target = target;
    ps.max_it = max_it;
    ps.status = KC_STATUS_MAX_CYCLES;
    ps.napp = 1;
    ps.hist = h->d_hist;
    KC_CUDA(h, cudaMemcpyAsync(h->d_pcg, &ps, sizeof(ps), cudaMemcpyHostToDevice, h->stream));
    KC_CUDA(h, cudaGraphLaunch(pg->exec, h->stream));
    KC_CUDA(h, cudaMemcpyAsync(&ps, h->d_pcg, sizeof(ps), cudaMemcpyDeviceToHost, h->stream));
    KC_CUDA(h, cudaStreamSynchronize(h->stream));
    it = ps.it;
    st = ps.status;
    napp = ps.napp;
    if (hist && it > 0) KC_CUDA(h, cudaMemcpy(hist + 1, h->d_hist + 1, sizeof(double) * it, cudaMemcpyDeviceToHost));
    for (int j = 1; j < h->n; ++j) {  // coarse levels are scratch after the cycles
      h->L[j].vzero = true;
      h->L[j].cur = 0;
    }
  } else {
    if ((rc = pcg_precondition(h, kappa, precond, ctx, hr, hz))) return rc;
    ++napp;
    if ((rc = red_dot(h, r, L0.v[L0.cur], 0, S_RZ, false))) return rc;
    KC_CUDA(h, cudaMemcpyAsync(h->p, L0.v[L0.cur], L0.elems * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
    if ((rc = fetch_scalars(h, S_MEAS + 1))) return rc;
    if (!(h->h_scal[S_RZ] > 0.0)) {
      st = KC_STATUS_BREAKDOWN;
    } else {
      for (it = 1; it <= max_it; ++it) {
        k_pcg_apply_dot2<<<grid2((m + 1) / 2, m, KC_RY), kBlock, 0, h->stream>>>(h->p, h->ap, m, P, L0.st,
                                                                              h->d_pcgpart);
        KC_LAUNCH_CHECK(h);
        k_red_final<false><<<1, KC_RED_THREADS, 0, h->stream>>>(h->d_pcgpart, KC_PCG_BLOCKS2(m), h->d_scal + S_PAP);
        KC_LAUNCH_CHECK(h);
        if (mx)
          k_pcg_update_xr<true><<<KC_RED_BLOCKS, KC_RED_THREADS, 0, h->stream>>>(h->x, r, h->p, h->ap, m, P, h->d_scal,
                                                                                  S_RZ, S_PAP, h->d_part, nullptr);
        else
          k_pcg_update_xr<false><<<KC_RED_BLOCKS, KC_RED_THREADS, 0, h->stream>>>(h->x, r, h->p, h->ap, m, P,
                                                                                   h->d_scal, S_RZ, S_PAP, h->d_part,
                                                                                   nullptr);
        KC_LAUNCH_CHECK(h);
        k_red_final<true><<<1, KC_RED_THREADS, 0, h->stream>>>(h->d_part, KC_RED_BLOCKS, h->d_scal + S_MEAS);
        KC_LAUNCH_CHECK(h);
        if ((rc = fetch_scalars(h, S_MEAS + 1))) return rc;
        if (!(h->h_scal[S_PAP] > 0.0)) {  // no measure at this step: NaN marks it
          st = KC_STATUS_BREAKDOWN;
          if (hist) hist[it] = NAN;
          break;
        }
        cur = h->h_scal[S_MEAS];
        if (hist) hist[it] = cur;
        if (cur <= target) {
          st = KC_STATUS_CONVERGED;
          break;
        }
        if ((rc = pcg_precondition(h, kappa, precond, ctx, hr, hz))) return rc;
        ++napp;
        if ((rc = red_dot(h, r, L0.v[L0.cur], 0, S_RZN, false))) return rc;
        k_pcg_update_p<<<KC_RED_BLOCKS, KC_RED_THREADS, 0, h->stream>>>(h->p, L0.v[L0.cur], m, P, h->d_scal, S_RZN,
                                                                       S_RZ);
        KC_LAUNCH_CHECK(h);
        k_copy_scalar<<<1, 32, 0, h->stream>>>(h->d_scal, S_RZ, S_RZN);
        KC_LAUNCH_CHECK(h);
        if ((rc = fetch_scalars(h, S_RZN + 1))) return rc;
        if (!(h->h_scal[S_RZN] > 0.0)) {
          st = KC_STATUS_BREAKDOWN;
          break;
        }
      }
      if (it > max_it) it = max_it;
    }
  }
  KC_CUDA(h, cudaEventRecord(h->ev1, h->stream));
  KC_CUDA(h, cudaEventSynchronize(h->ev1));
  float ms = 0.f;
  KC_CUDA(h, cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  if (device_ms) *device_ms = ms;
  if (x_out) {
    if ((rc = download_interior(h, x_out, h->x))) return rc;
    KC_CUDA(h, cudaStreamSynchronize(h->stream));
  }
  *iterations = it;
  *status = st;
  if (n_precond) *n_precond = napp;
  return KC_OK;
}

// ===========================================================================
// row-strip kernels (multi-GPU decomposition)
// ===========================================================================
namespace {
St9 strip_stencil(const double* w9, double omega) {
  St9 s{};
  for (int k = 0; k < 9; ++k) s.w[k] = std::fabs(w9[k]) <= DBL_EPSILON ? 0.0 : w9[k];  // ndimage tap drop
  s.center = w9[4];
  s.c = omega / s.center;
  return s;
}
int strip_err(cudaError_t e) {
  if (e == cudaSuccess) return KC_OK;
  g_create_err = cudaGetErrorString(e);
  return KC_ECUDA;
}
}  // namespace

extern "C" int kc_strip_jacobi(const double* u, const double* f, double* out, int ny, int nx, int pitch,
                               const double* w9, double omega, int zero_u, void* stream) {
  if (!f || !out || !w9 || ny < 0 || nx < 0) return KC_EINVAL;
  if (w9[4] == 0.0) return KC_EINVAL;
  if (ny == 0 || nx == 0) return KC_OK;
  dim3 g((nx + KSTR_BX - 1) / KSTR_BX, (ny + KSTR_BY - 1) / KSTR_BY);
  k_strip_jacobi<<<g, dim3(KSTR_BX, KSTR_BY), 0, (cudaStream_t)stream>>>(u, f, out, ny, nx, pitch,
                                                                        strip_stencil(w9, omega), zero_u);
  return strip_err(cudaGetLastError());
}

extern "C" int kc_strip_resid_restrict(const double* u, const double* f, double* fc, int ncy, int ncx, int pitch,
                                       int pitch_c, const double* w9, int zero_u, void* stream) {
  if (!f || !fc || !w9 || ncy < 0 || ncx < 0) return KC_EINVAL;
  if (ncy == 0 || ncx == 0) return KC_OK;
  dim3 g((ncx + KSTR_BX - 1) / KSTR_BX, (ncy + KSTR_BY - 1) / KSTR_BY);
  k_strip_resid_restrict<<<g, dim3(KSTR_BX, KSTR_BY), 0, (cudaStream_t)stream>>>(
      u, f, fc, ncy, ncx, pitch, pitch_c, strip_stencil(w9, 1.0), zero_u);
  return strip_err(cudaGetLastError());
}

extern "C" int kc_strip_prolong_add(double* v, const double* vc, int ny, int nx, int pitch, int pitch_c,
                                    int v_zero, void* stream) {
  if (!v || !vc || ny < 0 || nx < 0) return KC_EINVAL;
  if (ny == 0 || nx == 0) return KC_OK;
  dim3 g((nx + KSTR_BX - 1) / KSTR_BX, (ny + KSTR_BY - 1) / KSTR_BY);
  k_strip_prolong_add<<<g, dim3(KSTR_BX, KSTR_BY), 0, (cudaStream_t)stream>>>(v, vc, ny, nx, pitch, pitch_c, v_zero);
  return strip_err(cudaGetLastError());
}

extern "C" int kc_strip_norms(const double* v, const double* f, int ny, int nx, int pitch, const double* w9,
                              double* out, void* stream) {
  if (!v || !f || !out || !w9) return KC_EINVAL;
  static thread_local double* part = nullptr;  // per-thread scratch for the block partials
  const int nb = 1184;  // 8 blocks per SM: enough rows in flight to stream v and f
  if (!part) {
    cudaError_t e = cudaMalloc(&part, sizeof(double) * 2 * nb);
    if (e != cudaSuccess) return strip_err(e);
  }
  k_strip_norms<<<nb, 256, 0, (cudaStream_t)stream>>>(v, f, ny, nx, pitch, strip_stencil(w9, 1.0), part);
  k_strip_norms_final<<<1, 256, 0, (cudaStream_t)stream>>>(part, nb, out);
  return strip_err(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// device-side loops of the distributed solvers (kc_dist.cuh)
// ---------------------------------------------------------------------------
extern "C" int kc_strip_apply_dot(const double* p, double* ap, int ny, int nx, int pitch, const double* w9,
                                  double* part, double* scal, int slot, void* stream) {
  if (!p || !ap || !w9 || !part || !scal || ny < 0 || nx <= 0 || slot < 0 || slot >= KC_DS_SLOTS) return KC_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  k_strip_apply_dot<<<KDS_NB, 256, 0, s>>>(p, ap, ny, nx, pitch, strip_stencil(w9, 1.0), part, scal);
  k_dist_final<<<1, 256, 0, s>>>(part, KDS_NB, scal, slot);
  return strip_err(cudaGetLastError());
}

extern "C" int kc_strip_dot(const double* a, const double* b, int ny, int nx, int pitch, double* part, double* scal,
                            int slot, void* stream) {
  if (!a || !b || !part || !scal || ny < 0 || nx <= 0 || slot < 0 || slot >= KC_DS_SLOTS) return KC_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  k_strip_dot<<<KDS_NB, 256, 0, s>>>(a, b, ny, nx, pitch, part, scal);
  k_dist_final<<<1, 256, 0, s>>>(part, KDS_NB, scal, slot);
  return strip_err(cudaGetLastError());
}

extern "C" int kc_strip_pcg_update_xr(double* x, double* r, const double* p, const double* ap, int ny, int nx,
                                      int pitch, int measure_x, double* part, double* scal, void* stream) {
  if (!x || !r || !p || !ap || !part || !scal || ny < 0 || nx <= 0) return KC_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  k_strip_pcg_update_xr<<<KDS_NB, 256, 0, s>>>(x, r, p, ap, ny, nx, pitch, scal, measure_x, part);
  k_dist_final<<<1, 256, 0, s>>>(part, KDS_NB, scal, KC_DS_MEAS);
  return strip_err(cudaGetLastError());
}

extern "C" int kc_strip_pcg_update_p(double* p, const double* z, int ny, int nx, int pitch, const double* scal,
                                     void* stream) {
  if (!p || !z || !scal || ny < 0 || nx <= 0) return KC_EINVAL;
  k_strip_pcg_update_p<<<KDS_NB, 256, 0, (cudaStream_t)stream>>>(p, z, ny, nx, pitch, scal);
  return strip_err(cudaGetLastError());
}

extern "C" int kc_strip_residual(const double* x, const double* f, double* r, int ny, int nx, int pitch,
                                 const double* w9, void* stream) {
  if (!x || !f || !r || !w9 || ny < 0 || nx <= 0) return KC_EINVAL;
  k_strip_residual<<<KDS_NB, 256, 0, (cudaStream_t)stream>>>(x, f, r, ny, nx, pitch, strip_stencil(w9, 1.0));
  return strip_err(cudaGetLastError());
}

extern "C" int kc_strip_copy_if(const double* src, double* dst, int ny, int nx, int pitch, const double* scal,
                                void* stream) {
  if (!src || !dst || !scal || ny < 0 || nx <= 0) return KC_EINVAL;
  k_strip_copy_if<<<KDS_NB, 256, 0, (cudaStream_t)stream>>>(src, dst, ny, nx, pitch, scal);
  return strip_err(cudaGetLastError());
}

extern "C" int kc_dist_step(int kind, double* scal, double* hist, void* stream) {
  if (!scal || !hist || kind < KC_DS_PCG_RZ0 || kind > KC_DS_SOLVE) return KC_EINVAL;
  k_dist_step<<<1, 32, 0, (cudaStream_t)stream>>>(kind, scal, hist);
  return strip_err(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// fused strip passes: k_pre / k_post (kc_stream.cuh) on a row strip whose
// buffers carry `hb` halo rows (exchanged by the caller, depth >= nu+1 for
// the pre pass, >= nu for the post pass) -- two launches per routine call
// instead of nu + 2 per-op kernels, and two halo exchanges
// ---------------------------------------------------------------------------
namespace {
int strip_slots(const void* fn, int D) {
  static std::map<const void*, int> cache;
  static int sms = 0;
  auto it = cache.find(fn);
  if (it != cache.end()) return it->second;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ks_smem_bytes(D));
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, 128, ks_smem_bytes(D)) != cudaSuccess || blocks < 1)
    blocks = 1;
  return cache[fn] = blocks * 4 * sms;
}
// sym: shared stencil products as in ks_pre_fn / ks_post_fn (exact build
// only; the post pass keeps SYM <= 1)
int strip_sym(const double* w9, double omega) {
  static const int sym_max = getenv("KC_SYM") ? atoi(getenv("KC_SYM")) : (KC_FAST ? 0 : 2);
  return std::min(sym_max, ks_sym(strip_stencil(w9, omega)));
}
KsFn strip_pre_fn(int nu, bool zero, int sym = 0) {
  if (sym == 2 && nu == 2 && !zero) return k_pre<2, false, false, true, 2>;
  if (sym && nu == 2 && !zero) return k_pre<2, false, false, true, 1>;
#define KS_SPRE(N) return zero ? k_pre<N, true, false, true> : k_pre<N, false, false, true>
  switch (nu) {
    case 0: KS_SPRE(0);
    case 1: KS_SPRE(1);
    case 2: KS_SPRE(2);
    case 3: KS_SPRE(3);
    case 4: KS_SPRE(4);
  }
#undef KS_SPRE
  return nullptr;
}
KsFn strip_post_fn(int nu, bool vz, int sym = 0) {
  if (sym && nu == 2) return vz ? k_post<2, true, 0, true, 1> : k_post<2, false, 0, true, 1>;
#define KS_SPOST(N) return vz ? k_post<N, true, 0, true> : k_post<N, false, 0, true>
  switch (nu) {
    case 0: KS_SPOST(0);
    case 1: KS_SPOST(1);
    case 2: KS_SPOST(2);
    case 3: KS_SPOST(3);
    case 4: KS_SPOST(4);
  }
#undef KS_SPOST
  return nullptr;
}
StreamParams strip_params(int rows, int nx, int pitch, int pitch_c, int crows, int gy0, int mg, int hb, int hbc,
                          int qlo, int qhi, const double* w9, double omega, int D, const void* fn, int* nwarps) {
  StreamParams p{};
  p.m = nx;
  p.P = pitch;
  p.mc = (nx - 1) / 2;
  p.Pc = pitch_c;
  p.s = strip_stencil(w9, omega);
  p.rows = rows;
  p.gy0 = gy0;
  p.mg = mg;
  p.hb = hb;
  p.mcr = crows;
  p.hbc = hbc;
  p.qlo = qlo;
  p.qhi = qhi;
  p.nbands = (p.mc + 1 + ks_npb(D) - 1) / ks_npb(D);
  p.nq = ks_choose_nq(qhi - qlo - 1, p.nbands, strip_slots(fn, D));
  *nwarps = p.nbands * ((qhi - qlo + p.nq - 1) / p.nq);
  return p;
}
int floor2(int a) { return a >= 0 ? a / 2 : -((1 - a) / 2); }
// the fine input rows [*lo, *hi] (local) the owned outputs of a window
// [qlo, qhi) depend on; false: nothing owned
bool pre_window_rows(int rows, int crows, int nu1, int qlo, int qhi, int* lo, int* hi) {
  const int D = nu1 + 1;
  const int fe = std::min(2 * qhi, rows), ce = std::min(qhi, crows);  // owned fine rows end, coarse rows end
  const bool fine = nu1 > 0 && fe > 2 * qlo, coarse = ce > qlo;
  if (!fine && !coarse) return false;
  *lo = 2 * qlo - D;
  *hi = std::max(fine ? fe - 1 + nu1 : INT_MIN, coarse ? 2 * ce + D : INT_MIN);
  return true;
}
// post: fine input rows and coarse rows of vc
bool post_window_rows(int rows, int nu2, int qlo, int qhi, int* lo, int* hi, int* clo, int* chi) {
  const int fe = std::min(2 * qhi, rows);
  if (fe <= 2 * qlo) return false;
  *lo = 2 * qlo - nu2;
  *hi = fe - 1 + nu2;
  *clo = (*lo % 2 == 0) ? *lo / 2 - 1 : floor2(*lo);  // fine row 2q reads coarse rows q-1, q; 2q+1 reads q
  *chi = floor2(*hi);
  return true;
}
}  // namespace

extern "C" int kc_strip_pre(const double* u, const double* f, double* uo, double* fc, int rows, int nx, int pitch,
                            int pitch_c, int crows, int gy0, int mg, int hb, const double* w9, double omega, int nu1,
                            int zero_u, void* stream) {
  if (hb < nu1 + 2 || crows < 0) return KC_EINVAL;
  return kc_strip_pre_window(u, f, uo, fc, rows, nx, pitch, pitch_c, crows, gy0, mg, hb, 0, crows + 1, w9, omega, nu1,
                             zero_u, stream);
}

extern "C" int kc_strip_pre_window(const double* u, const double* f, double* uo, double* fc, int rows, int nx,
                                   int pitch, int pitch_c, int crows, int gy0, int mg, int hb, int q_lo, int q_hi,
                                   const double* w9, double omega, int nu1, int zero_u, void* stream) {
  if (!f || !uo || !fc || !w9 || rows < 1 || nx < 3 || crows < 0 || hb < 0 || gy0 < 0 || gy0 % 2) return KC_EINVAL;
  if (!zero_u && !u) return KC_EINVAL;
  if (nu1 < 0 || nu1 > 4 || (nu1 > 0 && w9[4] == 0.0)) return KC_EINVAL;
  if (q_lo < 0 || q_hi < q_lo || q_hi > crows + 1) return KC_EINVAL;
  int lo = 0, hi = 0;
  if (!pre_window_rows(rows, crows, nu1, q_lo, q_hi, &lo, &hi)) return KC_OK;  // nothing owned
  if (lo < -hb || hi > rows + hb - 1) return KC_EINVAL;  // the window reaches rows the buffers do not hold
  int nw = 0;
  KsFn fn = strip_pre_fn(nu1, zero_u != 0, strip_sym(w9, omega));
  StreamParams p = strip_params(rows, nx, pitch, pitch_c, crows, gy0, mg, hb, 1, q_lo, q_hi, w9, omega, nu1 + 1,
                                (const void*)fn, &nw);
  // the kernels index from the padded-array base: kc_idx(P, 0, 0) = P + KC_OX
  const ptrdiff_t ob = (ptrdiff_t)pitch + KC_OX, obc = (ptrdiff_t)pitch_c + KC_OX;
  p.u = u ? u - ob : nullptr;
  p.f = f - ob;
  p.uo = uo - ob;
  p.fc = fc - obc;
  fn<<<(nw + 3) / 4, 128, ks_smem_bytes(nu1 + 1), (cudaStream_t)stream>>>(p);
  return strip_err(cudaGetLastError());
}

extern "C" int kc_strip_post(const double* u, const double* f, double* uo, const double* vc, int rows, int nx,
                             int pitch, int pitch_c, int crows, int gy0, int mg, int hb, int hbc, const double* w9,
                             double omega, int nu2, int v_zero, void* stream) {
  if (hb < nu2 || hbc < nu2 / 2 + 1 || crows < 0) return KC_EINVAL;
  return kc_strip_post_window(u, f, uo, vc, rows, nx, pitch, pitch_c, crows, gy0, mg, hb, hbc, 0, crows + 1, w9,
                              omega, nu2, v_zero, stream);
}

extern "C" int kc_strip_post_window(const double* u, const double* f, double* uo, const double* vc, int rows,
                                    int nx, int pitch, int pitch_c, int crows, int gy0, int mg, int hb, int hbc,
                                    int q_lo, int q_hi, const double* w9, double omega, int nu2, int v_zero,
                                    void* stream) {
  if (!f || !uo || !vc || !w9 || rows < 1 || nx < 3 || crows < 0 || hb < 0 || hbc < 0 || gy0 < 0 || gy0 % 2)
    return KC_EINVAL;
  if (!v_zero && !u) return KC_EINVAL;
  if (nu2 < 0 || nu2 > 4 || (nu2 > 0 && w9[4] == 0.0)) return KC_EINVAL;
  if (q_lo < 0 || q_hi < q_lo || q_hi > crows + 1) return KC_EINVAL;
  int lo = 0, hi = 0, clo = 0, chi = 0;
  if (!post_window_rows(rows, nu2, q_lo, q_hi, &lo, &hi, &clo, &chi)) return KC_OK;
  if (lo < -hb || hi > rows + hb - 1 || clo < -hbc || chi > crows + hbc - 1) return KC_EINVAL;
  int nw = 0;
  KsFn fn = strip_post_fn(nu2, v_zero != 0, strip_sym(w9, omega));
  StreamParams p = strip_params(rows, nx, pitch, pitch_c, crows, gy0, mg, hb, hbc, q_lo, q_hi, w9, omega,
                                nu2 > 0 ? nu2 : 1, (const void*)fn, &nw);
  const ptrdiff_t ob = (ptrdiff_t)pitch + KC_OX, obc = (ptrdiff_t)pitch_c + KC_OX;  // see kc_strip_pre
  p.u = u ? u - ob : nullptr;
  p.f = f - ob;
  p.uo = uo - ob;
  p.vc = vc - obc;
  fn<<<(nw + 3) / 4, 128, ks_smem_bytes(nu2 > 0 ? nu2 : 1), (cudaStream_t)stream>>>(p);
  return strip_err(cudaGetLastError());
}

static int set_device(kc_handle* h, int level, int which, const double* dev, long long ny, long long nx,
                      long long pitch, bool sync) {
  if (!h || !dev) return KC_EINVAL;
  int rc = check_level(h, level);
  if (rc) return rc;
  Level& L = h->L[level - 1];
  if (ny != L.ny || nx != L.m) KC_FAIL(h, KC_EINVAL, "shape (%lld, %lld) != level %d shape (%d, %d)", ny, nx, level, L.ny, L.m);
  double* dst = which == KC_WHICH_F ? L.f : L.v[L.cur];
  KC_CUDA(h, cudaMemcpy2DAsync(dst + kc_idx(L.P, 0, 0), sizeof(double) * L.P, dev, sizeof(double) * pitch,
                               sizeof(double) * L.m, L.ny, cudaMemcpyDeviceToDevice, h->stream));
  if (sync) KC_CUDA(h, cudaStreamSynchronize(h->stream));
  if (which != KC_WHICH_F) L.vzero = false;
  return KC_OK;
}

static int get_device(kc_handle* h, int level, int which, double* dev, long long ny, long long nx, long long pitch,
                      bool sync) {
  if (!h || !dev) return KC_EINVAL;
  int rc = check_level(h, level);
  if (rc) return rc;
  Level& L = h->L[level - 1];
  if (ny != L.ny || nx != L.m) KC_FAIL(h, KC_EINVAL, "shape (%lld, %lld) != level %d shape (%d, %d)", ny, nx, level, L.ny, L.m);
  if (which != KC_WHICH_F && (rc = ex_materialize(h, level - 1))) return rc;
  const double* src = which == KC_WHICH_F ? L.f : L.v[L.cur];
  KC_CUDA(h, cudaMemcpy2DAsync(dev, sizeof(double) * pitch, src + kc_idx(L.P, 0, 0), sizeof(double) * L.P,
                               sizeof(double) * L.m, L.ny, cudaMemcpyDeviceToDevice, h->stream));
  if (sync) KC_CUDA(h, cudaStreamSynchronize(h->stream));
  return KC_OK;
}

extern "C" int kc_set_device(kc_handle* h, int level, int which, const double* dev, long long ny, long long nx,
                             long long pitch) {
  return set_device(h, level, which, dev, ny, nx, pitch, true);
}

extern "C" int kc_get_device(kc_handle* h, int level, int which, double* dev, long long ny, long long nx,
                             long long pitch) {
  return get_device(h, level, which, dev, ny, nx, pitch, true);
}

extern "C" int kc_set_device_async(kc_handle* h, int level, int which, const double* dev, long long ny,
                                   long long nx, long long pitch) {
  return set_device(h, level, which, dev, ny, nx, pitch, false);
}

extern "C" int kc_get_device_async(kc_handle* h, int level, int which, double* dev, long long ny, long long nx,
                                   long long pitch) {
  return get_device(h, level, which, dev, ny, nx, pitch, false);
}

extern "C" int kc_set_stream(kc_handle* h, void* stream) {
  if (!h) return KC_EINVAL;
  // NULL is CUDA's stream 0 (the legacy default stream), (void*)-1 the handle's own
  h->stream = stream == (void*)-1 ? h->own_stream : (cudaStream_t)stream;
  return KC_OK;
}

// One kappa-cycle issued op by op on the handle's stream, nothing awaited:
// capturable into a caller's CUDA graph (the bottom schedules and occupancy
// tables are built on first use, so run it once outside a capture first).
extern "C" int kc_cycle_enqueue(kc_handle* h, int kappa) {
  if (!h) return KC_EINVAL;
  if (kappa < 1) KC_FAIL(h, KC_EINVAL, "cycle counter must be >= 1, got %d", kappa);
  if (kappa > h->n) kappa = h->n;
  std::vector<Op> ops;
  flatten(h, 0, kappa, ops);
  for (const Op& op : ops) {
    const int rc = ex_op(h, op);
    if (rc) return rc;
  }
  return KC_OK;
}
