// kc_bottom.cuh — persistent kernel for the latency-bound bottom of the
// hierarchy: a 16-CTA thread-block cluster entering at
// side <= 255 (see below), or one CTA entering at side <= 63.
//
// Every remaining level (v ping-pong pair and f, each with its zero ghost
// ring) lives in shared memory.  The kernel loads f (and v unless it is the
// zero guess) of the entry level from HBM, replays the reference's
// kappa_cycle recursion (cycle.py:204-220) from a host-built phase list, and
// writes v back.  Every routine call of the bottom levels costs barriers
// instead of kernel launches, so host-visible launches per cycle no longer
// grow with kappa's polynomial call count.
//
// Design for latency (measured on B200, tools/micro: fp64 dependent op 8
// cycles, __syncthreads 47-115, __syncwarp 31, a bare 3x3 Jacobi phase ~340,
// cluster barrier ~490 / ~940 with remote stores outstanding):
//  * one control loop replays one phase descriptor per iteration at a single
//    inlined site, so the kernel stays small; 384 threads per CTA (exact
//    build; 256 in the FMA build, see KC_BOT_THREADS) leave 170 registers
//    per thread (the loop is register-bound: 512 threads spilled);
//  * the warps that work on a level scale with its size: all for sides
//    >= 31 (CTA or cluster barrier), 8 for 15 (named barrier), 1-2 for the
//    smallest (__syncwarp / named barrier), and idle warps skip the phase;
//    whole frames on sides <= 15 run as one descriptor (PH_TINY);
//  * stencil phases are register-blocked 4 rows per thread (3 new loads per
//    row instead of 9) where there are enough rows;
//  * the coarsest 1x1 solve is folded into its parent's restriction.
// Per-point arithmetic is identical to the HBM kernels (kc_common.cuh), so
// iterates stay bit-identical to the reference.  The redundant second
// coarsest solve under level n-1 (cycle.py:7-10) recomputes the identical
// f/center and is skipped; CycleStats still counts it.
#pragma once
#include <cooperative_groups.h>
#include "kc_common.cuh"

// Two launch shapes, one kernel:
//  * single CTA (entry side <= KC_BOT_MAX_M): every level in its shared
//    memory, as described above;
//  * thread-block cluster of cs CTAs (16, non-portable; 8 as a fallback)
//    entering at a side <= KC_CLU_MAX_M (255): the levels with side >=
//    KC_CLU_MIN_STRIP (31) are split into row strips of R = (m+1)/cs rows,
//    one per CTA, each with one halo row above and below.  A strip phase is
//    run by every CTA on its own rows; outputs on a strip's first/last row
//    are also stored into the neighbour's halo row through distributed
//    shared memory (st to a mapa'd address), and the phase ends with a
//    cluster barrier (release/acquire), so the next phase sees them.
//    Coarser levels live in CTA 0 only and run as in the single-CTA case
//    while the other CTAs wait at the next cluster barrier (PH_CSYNC);
//    the restriction into them and the prolongation out of them read and
//    write CTA 0's shared memory remotely.  The full-coarsening strips nest
//    (coarse strip = fine strip / 2), so every transfer is strip-local.
// Measured (tools/micro/clsync): a 16-CTA cluster barrier costs ~490
// cycles, ~940 with remote stores outstanding — cheaper than one graph
// kernel node (~1.1 us) and far cheaper than the 255^2 / 127^2 levels on
// the graph's tile kernels.
#define KC_BOT_MAX_M 63
#define KC_CLU_MAX_M 255
#ifndef KC_CLU_ENTRY_M
#define KC_CLU_ENTRY_M 127  // default entry (kc_engine.cu)
#endif
#ifndef KC_CLU_MIN_STRIP
#define KC_CLU_MIN_STRIP 63  // coarser levels are replicated in every CTA (31^2: 1.1 k vs 1.9 k cycles per phase)
#endif
#define KC_BOT_MAXLEV 8
#ifndef KC_BOT_THREADS
// FMA build: 8 warps, up to 255 registers without spills (at 384 threads the
// frame-operator and pair paths spill at the 168-register cap: n=12 kappa=3
// cycle 0.889 vs 0.845 ms); exact build (interpreter frames): 12 warps
// (256 threads: 1.148 -> 1.206 ms)
#if KC_FAST
#define KC_BOT_THREADS 256
#else
#define KC_BOT_THREADS 384
#endif
#endif
#define KC_BOT_WARPS (KC_BOT_THREADS / 32)
#define KC_BOT_RB 4  // rows per thread in stencil phases

#define KC_BOT_MAXPH 1024  // phase descriptors per launch (host-checked; a W sub-cycle from 127^2 needs < 300)

// per-level constants, computed on the host (bot_geometry; the strip rows
// of each rank are finished on the device) and kept in shared memory: each
// phase reads a few LDS.128 instead of doing address math
struct BotLv {
  int m, S, vo0, vo1;           // side, stride, smem offsets of the v buffers (interior origin)
  int fo, nitem1, nitem4, rows;  // f offset, stencil items for RB = 1 / 4, own interior rows
  int a, R, rb4, crows;          // first global row, strip height, RB = 4?, own rows of the child
  float inv, invc, invn;         // 1/m, 1/m_child, 1/(m_child+1)
  int mc;                        // child side
  int hb;                        // halo rows each side (1; KC_DEEP_HB on the deep-halo strip level)
};

#define KC_MV_M 15
#define KC_MV_N (KC_MV_M * KC_MV_M)  // 225 unknowns of a side-15 level
#define KC_MV_LD 226                 // row stride (16-byte multiple: cp.async)
// blocks: (k - 1) * 2 + {0: A_k, 1: B_k} for k = 1..3, then the PAIR
// operators P = A_kb B_ka + B_kb of the two frames a side-31 call makes from
// a zero guess, counters (ka, kb) = (2, 1), (3, 2), (3, 3): one
// matrix-vector phase instead of two (BotFrame31::frame)
#define KC_MV_PAIR0 6
#define KC_MV_NBLK 9
__host__ __device__ __forceinline__ int kc_mv_pair(int kap) {  // kap >= 2: the pair block of frames (kap, kap - 1)
  return kap == 2 ? KC_MV_PAIR0 : (kap == 3 ? KC_MV_PAIR0 + 1 : KC_MV_PAIR0 + 2);
}

struct BotParams {
  int nlev;  // levels resident in smem: entry level .. coarsest
  St9 st[KC_BOT_MAXLEV];
  double* gv;        // entry-level v in HBM (padded, pitch gP): read unless v_zero, always written
  const double* gf;  // entry-level f in HBM
  int gP;
  int v_zero;        // entry-level v is the zero guess
  const unsigned* sched;  // host-built phase list (bot_schedule), device memory
  int nsched;
  int final_cur;     // buffer holding the entry level's v after the schedule
  int nu1, nu2;      // sweeps inside PH_TINY frames
  int nstrip;        // leading levels split into row strips over the cluster (0: single CTA)
  int total;         // shared-memory doubles of all levels (bot_smem_doubles)
  int deep;          // the deep-halo strip level (PH_FRAME63), or -1
  int deep0;         // the entry level has deep halos too and launches run as PH_FRAME127
  BotLv lv[KC_BOT_MAXLEV];  // bot_geometry (rank 0's strip rows)
  // side-15 frame operators (KC_FAST cluster launches; see "Frame operators"
  // below): blocks (kap - 1) * 2 + part of [A_kap | B_kap], 225 x KC_MV_LD
  // rows in global memory; the blocks this launch uses (mv_copy, a subset
  // of the handle's resident set) are copied row-sliced into every CTA's
  // shared memory at mv_off, slot mv_slot[block]
  const double* mv_mats;
  int mv_copy, mv_off, mv_rows, mv_xin;  // mv_xin: 2 x 225 doubles of packed inputs
  int mv_avail;      // blocks that exist (resident or read from global memory): frames use them
  int mv_slot[KC_MV_NBLK];
  // st.async phases (jitter builds: a runtime switch within the compile-time
  // KC_MV_ASYNC / KC_RB_ASYNC): bit 0 the frame-operator outputs, bit 1 the
  // 63^2 -> 31^2 broadcast
  int async;
};

// Frame operators (FMA build, cluster launches only).  A kappa_cycle frame on
// the side-15 level (with its 7^2, 3^2 and 1x1 children; BotTiny below) is a
// LINEAR map of its inputs: v_out = A_k v_in + B_k f (v_in = 0 on a zero
// guess), A_k, B_k fixed 225 x 225 matrices for frame counter k (k >= 3 is
// the W frame at this depth: kappa_cycle(15, k) recurses into 7^2 with
// counters k, k - 1 >= 2, which are W there).  The engine builds the columns
// on the device by running the very same frame code on unit inputs
// (k_tiny_mats), each CTA of the 16-CTA cluster keeps a row slice of the
// needed blocks in its shared memory, and a frame becomes one cluster-wide
// matrix-vector phase (bot_mv_frame): ~2 k cycles instead of the ~10-12 k
// of 30+ barrier-separated tiny phases.  The side-15 level is replicated in
// every CTA like all non-strip levels (BotBuilder), so a frame reads its
// inputs locally and stores its rows into every CTA's copy.  A frame whose
// blocks are not resident runs the interpreter on every CTA's copy.  The product rounds
// differently from the frame's own operation sequence, so this is FAST-only
// (the exact build keeps the frames); parity bar as for the FMA build.

// smem geometry of level d (entry side m0): side m_d = ((m0+1) >> d) - 1,
// stride S = m+2, three arrays v0, v1, f of (rows+2) x S, rows = m, or the
// strip height R = (m+1)/cs for the first nstrip levels (same on every CTA,
// so a local address maps to the same array on any rank).
__host__ __device__ __forceinline__ int bot_m(int m0, int d) { return ((m0 + 1) >> d) - 1; }
__host__ __device__ __forceinline__ int bot_rows(int m0, int d, int nstrip, int cs) {
  return d < nstrip ? (bot_m(m0, d) + 1) / cs : bot_m(m0, d);
}
// halo rows each side of level d: KC_DEEP_HB on the deep-halo strip level
// (PH_FRAME63 computes its stages on the halo rows redundantly), else 1
#define KC_DEEP_HB 4
__host__ __device__ __forceinline__ int bot_hb(int d, int deep, int deep0 = 0) {
  return (d == deep || (deep0 && d == 0)) ? KC_DEEP_HB : 1;
}
__host__ __device__ __forceinline__ int bot_off(int m0, int d, int nstrip = 0, int cs = 1, int deep = -1,
                                                int deep0 = 0) {
  int off = 0;
  for (int j = 0; j < d; ++j) {
    const int s = bot_m(m0, j) + 2;
    off += 3 * (bot_rows(m0, j, nstrip, cs) + 2 * bot_hb(j, deep, deep0)) * s;
  }
  return off;
}
__host__ __device__ __forceinline__ int bot_smem_doubles(int m0, int nlev, int nstrip = 0, int cs = 1,
                                                         int deep = -1, int deep0 = 0) {
  return bot_off(m0, nlev, nstrip, cs, deep, deep0);
}
__host__ __device__ __forceinline__ int bot_warps(int m) {
  return m >= 31 ? KC_BOT_WARPS : (m >= 15 ? 8 : 1);  // 2 warps at m = 7 measured slower
}

// Per-level geometry of a launch (host; m0 = entry side, cs = cluster size):
// what the kernel used to derive with integer divisions in its prologue.
inline void bot_geometry(BotParams& bp, int m0, int cs) {
  const int nlev = bp.nlev, nstrip = bp.nstrip;
  bp.total = bot_smem_doubles(m0, nlev, nstrip, cs, bp.deep, bp.deep0);
  for (int d = 0; d < nlev; ++d) {
    const bool strip = d < nstrip;
    const int hb = bot_hb(d, bp.deep, bp.deep0);
    const int m = bot_m(m0, d), S = m + 2, base = bot_off(m0, d, nstrip, cs, bp.deep, bp.deep0);
    const int R = bot_rows(m0, d, nstrip, cs);
    const int mc = d + 1 < nlev ? bot_m(m0, d + 1) : 1;
    BotLv L{};
    L.m = m;
    L.S = S;
    L.R = R;
    L.mc = mc;
    L.a = 0;
    L.rows = strip ? (R < m ? R : m) : m;
    L.hb = hb;
    L.vo0 = base + hb * S + 1;
    L.vo1 = base + (R + 2 * hb) * S + hb * S + 1;
    L.fo = base + 2 * (R + 2 * hb) * S + hb * S + 1;
    L.nitem1 = L.rows * m;
    L.nitem4 = m * ((L.rows + 3) / 4);
    // RB = 4 where a thread would otherwise run more than one item: a full
    // 4-row item is four independent chains, little longer than one
    L.rb4 = strip ? (L.nitem1 > KC_BOT_THREADS) : (m >= 31);
    L.crows = strip ? ((mc < L.rows / 2) ? mc : L.rows / 2) : mc;
    L.inv = 1.0f / (float)m;
    L.invc = 1.0f / (float)mc;
    L.invn = 1.0f / (float)(mc + 1);
    bp.lv[d] = L;
  }
}

// Schedule perturbation (race testing; compute-sanitizer is closed on this
// pool): the KC_BOT_JITTER builds (libkcb200*_jitter.so, tests only) make
// about one warp in four sleep up to KC_BOT_JITTER ns right after every
// barrier, so a missing barrier between a stage that writes data and one
// that reads it (in this CTA or, through DSMEM, in another) shows up as a
// wrong, non-reproducible result (tests/test_gpu_jitter.py).
#ifdef KC_BOT_JITTER
__device__ __forceinline__ void bot_jitter() {
  unsigned h = (unsigned)clock64() ^ (blockIdx.x * 0x9E3779B9u) ^ ((threadIdx.x >> 5) * 0x85EBCA6Bu);
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  h = __shfl_sync(0xffffffffu, h, 0);  // warp-uniform
  if ((h & 3u) == 0u) __nanosleep(h % KC_BOT_JITTER);
}
#else
__device__ __forceinline__ void bot_jitter() {}
#endif
// a CTA barrier of the bottom kernel (with the jitter of the test builds)
__device__ __forceinline__ void bot_bar() {
  __syncthreads();
  bot_jitter();
}
__device__ __forceinline__ void bot_sync(int g) {
  if (g == KC_BOT_WARPS) bot_bar();
  else if (g == 1) __syncwarp();
  else if (g == 8) asm volatile("bar.sync 1, 256;" ::: "memory");
  else asm volatile("bar.sync 2, 64;" ::: "memory");
  bot_jitter();
}
// every thread of every CTA of the cluster; orders the DSMEM stores before it
__device__ __forceinline__ void clu_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  bot_jitter();
}

#ifdef KC_BOT_TRACE
__device__ long long kc_bot_trace[KC_BOT_TRACE];
__device__ int kc_bot_trace_op[KC_BOT_TRACE];
__device__ int kc_bot_trace_n;
__device__ long long kc_bot_trace_end[KC_BOT_TRACE];
// sub-phase stamps inside the compiled frames (tools/micro/bottrace.cu):
// CTA 0, thread 0, a code per point of BotDeep::run
__device__ long long kc_bot_sub[KC_BOT_TRACE];
__device__ int kc_bot_sub_code[KC_BOT_TRACE];
__device__ int kc_bot_sub_n;
#define KC_BOT_SUB(code)                                                      \
  do {                                                                        \
    if (threadIdx.x == 0 && blockIdx.x == 0 && kc_bot_sub_n < KC_BOT_TRACE) { \
      kc_bot_sub[kc_bot_sub_n] = clock64();                                   \
      kc_bot_sub_code[kc_bot_sub_n++] = (code);                               \
    }                                                                         \
  } while (0)
__device__ unsigned long long kc_bot_stamp[8];  // globaltimer: start, init, entry, phases, end (CTA 0)
__device__ __forceinline__ void kc_bot_mark(int k) {
  if (threadIdx.x == 0 && cooperative_groups::this_cluster().block_rank() == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    kc_bot_stamp[k] = t;
  }
}
#define KC_BOT_MARK(k) kc_bot_mark(k)
#else
#define KC_BOT_MARK(k)
#define KC_BOT_SUB(code) \
  do {                   \
  } while (0)
#endif

// Phase kinds (host-built list, BotBuilder below):
//   PH_JACOBI / PH_RESID / PH_RESTRICT / PH_PROLONG  one protocol routine;
//   PH_J2Z  two sweeps from the zero guess: u1 = 0 + c f is pointwise, so the
//           second sweep recomputes it at its 3x3 neighbours from f (+0.0 on
//           the ghost ring, exactly the Dirichlet value) -- same per-point
//           arithmetic, so results stay bit-identical;
//   PH_TINY a whole kappa_cycle frame on a level of side <= 15 (with its
//           children) run without interpreter overhead between its phases
//           (BotTiny below);
//   PH_JOIN gather a larger warp group; PH_CSYNC cluster barrier.
// (Residual+restriction and prolongation+sweep fusions for the small levels
// were measured slower -- larger kernel, longer dependent chains -- and the
// tiny frames replaced them.)
enum BotOp {
  PH_JACOBI = 0, PH_RESID = 1, PH_RESTRICT = 2, PH_PROLONG = 3, PH_JOIN = 4, PH_J2Z = 5, PH_TINY = 8, PH_CSYNC = 9,
  PH_FRAME31 = 10,  // a whole kappa_cycle frame on the replicated side-31 level (BotFrame31)
  PH_FRAME63 = 11,  // the pair of calls (kappa, kappa - 1) on the deep-halo side-63 strips (BotDeep)
  PH_FRAME127 = 12  // the whole launch: the 127^2 pair from a zero guess, deep halos on 127^2 and 63^2 (BotDeep)
};
#ifndef KC_BOT_TINY_M
#define KC_BOT_TINY_M 15  // frames on sides <= this run as PH_TINY (side 15 on 8 warps)
#endif
// Descriptor: bits 0-3 op, 4-6 level d, 7 src buffer, 8 zero guess, 9 child
// buffer (prolong), 10 child is the 1x1 coarsest (restrict), 11-12 warp
// group code, 13-16 cycle counter (PH_TINY), 17 strip phase (all CTAs).
//   PH_CSYNC  cluster barrier before a strip phase that follows CTA-0 work.
__host__ __device__ __forceinline__ unsigned bot_desc(int op, int d, int src, int zero, int cbuf, int cc, int g,
                                                      int kap = 0) {
  const unsigned gc = g >= KC_BOT_WARPS ? 3u : (g >= 8 ? 2u : (g >= 2 ? 1u : 0u));
  return (unsigned)op | ((unsigned)d << 4) | ((unsigned)src << 7) | ((unsigned)zero << 8) | ((unsigned)cbuf << 9) |
         ((unsigned)cc << 10) | (gc << 11) | ((unsigned)(kap > 15 ? 15 : kap) << 13);
}
__device__ __forceinline__ int bot_desc_g(unsigned e) {
  const unsigned gc = (e >> 11) & 3u;
  return gc == 3u ? KC_BOT_WARPS : (gc == 2u ? 8 : (gc == 1u ? 2 : 1));
}
#define BD_OP(e) ((int)((e) & 15u))
#define BD_D(e) ((int)(((e) >> 4) & 7u))
#define BD_SRC(e) ((int)(((e) >> 7) & 1u))
#define BD_ZERO(e) ((int)(((e) >> 8) & 1u))
#define BD_CBUF(e) ((int)(((e) >> 9) & 1u))
#define BD_CC(e) ((int)(((e) >> 10) & 1u))
#define BD_KAP(e) ((int)(((e) >> 13) & 15u))
#define BD_STRIP_BIT (1u << 17)

#include <vector>
// Flatten kappa_cycle over the smem-resident levels (cycle.py:204-220) into
// the bottom kernel's phase list (kc_bottom.cuh), tracking ping-pong buffers
// and zero guesses exactly like the executor does for the HBM levels.
struct BotBuilder {  // host side
  int m0, nlev, nu1, nu2;
  int nstrip = 0;           // levels d < nstrip are strip phases (all CTAs of the cluster)
  unsigned cur = 0, vz = 0;
  int gprev = KC_BOT_WARPS;
  bool fuse = true;         // emit PH_J2Z
  bool tiny = true;         // whole frames on sides <= KC_BOT_TINY_M as PH_TINY
  bool dry = false;         // track buffers only (inside a PH_TINY frame)
  unsigned mv_mask = 0;     // resident frame-operator blocks (0: frame operators off)
  unsigned mv_used = 0;     // blocks the emitted frames use (BotParams::mv_copy)
  int mv_last = -1;         // buffer the previous frame operator wrote
  bool mv_sync = false;     // an interpreter frame ran since: barrier before the next operator
  std::vector<unsigned> out;
  // Strip phases run on every CTA on its rows and end with a cluster
  // barrier.  Every coarser level is REPLICATED: each CTA holds all of it and
  // runs its phases on its own copy (group barrier only), so no phase reads
  // another CTA's copy and no cluster barrier is needed below the strips;
  // data enters the replicas by broadcast stores (the restriction out of the
  // last strip level, the frame operators' outputs), each followed by a
  // cluster barrier.
  void emit(int op, int d, int src, int zero, int cbuf, int cc, int kap = 0) {
    if (dry) return;
    if (d < nstrip) {
      gprev = KC_BOT_WARPS;  // a strip phase ends with a cluster barrier
      out.push_back(bot_desc(op, d, src, zero, cbuf, cc, KC_BOT_WARPS, kap) | BD_STRIP_BIT);
      return;
    }
    const int g = (op == PH_TINY && bot_m(m0, d) == 7) ? 2 : bot_warps(bot_m(m0, d));
    if (g > gprev) out.push_back(bot_desc(PH_JOIN, 0, 0, 0, 0, 0, g));
    gprev = g;
    out.push_back(bot_desc(op, d, src, zero, cbuf, cc, g, kap));
  }
  void relax(int d, int count) {
    int i = 0;
    if (fuse && count >= 2 && ((vz >> d) & 1u)) {  // two sweeps from the zero guess: result in buffer cur
      emit(PH_J2Z, d, (cur >> d) & 1u, 1, 0, 0);
      vz &= ~(1u << d);
      i = 2;
    }
    for (; i < count; ++i) {
      emit(PH_JACOBI, d, (cur >> d) & 1u, (vz >> d) & 1u, 0, 0);
      vz &= ~(1u << d);
      cur ^= 1u << d;
    }
  }
  bool frame31 = true;      // whole side-31 frames as PH_FRAME31 (replicated levels)
  int deep = -1;            // the deep-halo strip level: its call pairs as PH_FRAME63
  bool deep0 = false;       // deep halos on the entry level too: a zero-guess pair as PH_FRAME127
  // the launch's calls on the entry level: (k1) and, if k2 > 0, (k2)
  void top(int k1, int k2) {
    if (deep0 && !dry && (vz & 1u) && (k2 == k1 - 1 || (k1 == 1 && k2 == 0))) {
      // one descriptor for the whole launch; the dry replay follows BotDeep
      emit(PH_FRAME127, 0, cur & 1u, 1, 0, 0, k1);
      dry = true;
      rec(0, k1);
      if (k2 > 0) rec(0, k2);
      dry = false;
      return;
    }
    rec(0, k1);
    if (k2 > 0) rec(0, k2);
  }
  void rec(int d, int kap) {
    if (frame31 && fuse && !dry && d >= nstrip && bot_m(m0, d) == 31 && d + 5 == nlev && kap <= 15) {
      // one descriptor for the frame and everything below it; the dry replay
      // below follows BotFrame31 (and the frame-operator bookkeeping)
      emit(PH_FRAME31, d, (cur >> d) & 1u, (vz >> d) & 1u, 0, 0, kap);
      dry = true;
      rec(d, kap);
      dry = false;
      return;
    }
    if (mv_mask && d >= nstrip && bot_m(m0, d) == KC_MV_M && d < nlev - 1) {
      // frame operator: one cluster-wide phase (every CTA its rows, outputs
      // broadcast into every replica).  The output buffer alternates from
      // frame to frame, so it is never the one a slower CTA may still be
      // prolongating from (the previous frame's output); a continuing frame
      // (not a zero guess) reads that previous output and writes the other.
      // In a dry replay (inside PH_FRAME31) only the bookkeeping runs.
      const int k3 = kap < 3 ? kap : 3;
      const int z = (vz >> d) & 1u;
      const unsigned need = (1u << ((k3 - 1) * 2 + 1)) | (z ? 0u : (1u << ((k3 - 1) * 2)));
      if ((mv_mask & need) == need) {
        const int src = (cur >> d) & 1u;
        const int ob = z ? (mv_last >= 0 ? mv_last ^ 1 : src ^ 1) : src ^ 1;
        if (!dry) {
          if (mv_sync) out.push_back(bot_desc(PH_CSYNC, 0, 0, 0, 0, 0, KC_BOT_WARPS));
          gprev = KC_BOT_WARPS;
          out.push_back(bot_desc(PH_TINY, d, src, z, ob, 0, KC_BOT_WARPS, k3) | BD_STRIP_BIT);
        }
        mv_sync = false;
        mv_used |= need;
        mv_last = ob;
        cur = (cur & ~(1u << d)) | ((unsigned)ob << d);
        vz &= ~(1u << d);
        return;
      }
      mv_sync = true;  // interpreter frame below (every CTA on its replica)
      if (dry) {  // BotTiny's buffer rules (J2Z on)
        const bool t = tiny;
        tiny = false;
        rec_plain(d, kap);
        tiny = t;
        return;
      }
    }
    if (tiny && fuse && !dry && d >= nstrip && bot_m(m0, d) <= KC_BOT_TINY_M && d < nlev - 1 && kap <= 15) {
      // one descriptor; bot_tiny follows the rules below (J2Z on), so
      // replay them dry to track the buffers of level d
      emit(PH_TINY, d, (cur >> d) & 1u, (vz >> d) & 1u, 0, 0, kap);
      dry = true;
      rec(d, kap);
      dry = false;
      return;
    }
    rec_plain(d, kap);
  }
  void rec_plain(int d, int kap) {
    relax(d, nu1);
    const int c = (cur >> d) & 1u;
    const int z = (vz >> d) & 1u;
    const int cc = (d + 1 == nlev - 1);
    if (!z) emit(PH_RESID, d, c, 0, 0, 0);  // residual into buffer c^1
    emit(PH_RESTRICT, d, c ^ 1, z, 0, cc);
    cur &= ~(1u << (d + 1));
    if (cc) {
      vz &= ~(1u << (d + 1));  // both coarsest calls: one f/center inside the restriction
    } else {
      vz |= 1u << (d + 1);
      if (d + 1 == deep && !dry) {
        // both calls on the deep-halo level as one descriptor (every CTA);
        // the dry replay follows BotFrame63, which follows these rules
        emit(PH_FRAME63, d + 1, (cur >> (d + 1)) & 1u, 1, 0, 0, kap);
        dry = true;
        rec(d + 1, kap);
        if (kap > 1) rec(d + 1, kap - 1);
        dry = false;
      } else if (dry && kap > 1 && bot_m(m0, d) == 31 && bot_m(m0, d + 1) == KC_MV_M &&
                 ((mv_mask >> kc_mv_pair(kap)) & 1u)) {
        // inside BotFrame31: the pair operator of frames (kap, kap - 1) from
        // the zero guess, one matrix-vector phase (its buffer rule is a zero
        // frame's)
        const int src = (cur >> (d + 1)) & 1u;
        const int ob = mv_last >= 0 ? mv_last ^ 1 : src ^ 1;
        mv_sync = false;
        mv_used |= 1u << kc_mv_pair(kap);
        mv_last = ob;
        cur = (cur & ~(1u << (d + 1))) | ((unsigned)ob << (d + 1));
        vz &= ~(1u << (d + 1));
      } else {
        rec(d + 1, kap);
        if (kap > 1) rec(d + 1, kap - 1);
      }
    }
    emit(PH_PROLONG, d, (cur >> d) & 1u, (vz >> d) & 1u, (cur >> (d + 1)) & 1u, 0);
    vz &= ~(1u << d);
    relax(d, nu2);
  }
};


// y = i / m for i < 2^12, m <= 64: float reciprocal, exact for these ranges
__device__ __forceinline__ int bot_div(int i, float inv) { return (int)(((float)i + 0.5f) * inv); }

// Halo pushes of a strip phase: values on own rows 0 .. hb-1 also go to the
// upper neighbour's rows R .. R+hb-1 (its halo below), values on own rows
// R-hb .. R-1 to the lower neighbour's rows -hb .. -1 (hb = the level's halo
// depth).  Null for CTA-local levels and at the strip ends.
struct BotPush {
  double* up;  // upper neighbour's row R (row y of this CTA -> its row R + y)
  double* dn;  // lower neighbour's row 0 shifted by -R rows (row y -> its row y - R)
  int lo, hi;  // rows y < lo go up, rows y >= hi go down
  __device__ __forceinline__ void put(double* o, int S, int y, int x, double v) const {
    o[y * S + x] = v;
    if (up && y < lo) up[y * S + x] = v;
    if (dn && y >= hi) dn[y * S + x] = v;
  }
};
__device__ __forceinline__ BotPush bot_push(double* origin, const BotLv& L, bool strip, int rank, int cs) {
  BotPush p{nullptr, nullptr, 0, 1 << 30};
  if (strip) {
    cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
    if (rank > 0) p.up = cl.map_shared_rank(origin, rank - 1) + L.R * L.S;
    if (rank + 1 < cs) p.dn = cl.map_shared_rank(origin, rank + 1) - L.R * L.S;
    p.lo = L.hb;
    p.hi = L.R - L.hb;
  }
  return p;
}

// Jacobi sweep (zero guess folded) or residual on the rows x m block of a
// level (all of it, or this CTA's strip).  RB rows per item share their
// loads (3 new loads per row).
template <int RB>
__device__ __forceinline__ void bot_stencil(bool jac, bool zero, const double* __restrict__ u, double* __restrict__ o,
                                            const double* __restrict__ f, int m, int rows, int S, float inv,
                                            const St9& st, int tid, int nth, int nitems, const BotPush& ps) {
  for (int it = tid; it < nitems; it += nth) {
    const int rb = bot_div(it, inv);  // it / m
    const int x = it - rb * m;
    const int y0 = rb * RB;
    if (jac && zero) {
#pragma unroll
      for (int k = 0; k < RB; ++k)
        if (y0 + k < rows) ps.put(o, S, y0 + k, x, kc_jacobi_zero(f[(y0 + k) * S + x], st.c));
      continue;
    }
    const double* pu = u + y0 * S + x;
    if (RB > 1 && y0 + RB <= rows) {
      // full item: every load first, then RB independent chains (the
      // guarded loop below keeps the compiler from overlapping its rows)
      double w[RB + 2][3], fv[RB], out[RB];
#pragma unroll
      for (int k = 0; k < RB + 2; ++k)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) w[k][dx] = pu[(k - 1) * S + dx - 1];
#pragma unroll
      for (int k = 0; k < RB; ++k) fv[k] = f[(y0 + k) * S + x];
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const double au = kc_sum9(st, w[k][0], w[k][1], w[k][2], w[k + 1][0], w[k + 1][1], w[k + 1][2],
                                  w[k + 2][0], w[k + 2][1], w[k + 2][2]);
        out[k] = jac ? kc_jacobi_pt(w[k + 1][1], fv[k], au, st.c) : DSUB(fv[k], au);
      }
#pragma unroll
      for (int k = 0; k < RB; ++k) ps.put(o, S, y0 + k, x, out[k]);
      continue;
    }
    double a0 = pu[-S - 1], a1 = pu[-S], a2 = pu[-S + 1];
    double b0 = pu[-1], b1 = pu[0], b2 = pu[1];
#pragma unroll
    for (int k = 0; k < RB; ++k) {
      if (y0 + k < rows) {
        const double* pn = pu + (k + 1) * S;
        const double c0 = pn[-1], c1 = pn[0], c2 = pn[1];
        const int i = (y0 + k) * S + x;
        const double au = kc_sum9(st, a0, a1, a2, b0, b1, b2, c0, c1, c2);
        ps.put(o, S, y0 + k, x, jac ? kc_jacobi_pt(b1, f[i], au, st.c) : DSUB(f[i], au));
        a0 = b0; a1 = b1; a2 = b2;
        b0 = c0; b1 = c1; b2 = c2;
      }
    }
  }
}

// u2 = J(J(0)) into u, with u1 = 0 + c f recomputed at the neighbours (PH_J2Z)
__device__ __forceinline__ double bot_j2z_pt(const double* __restrict__ pf, int S, const St9& st) {
  double n1[9];
#pragma unroll
  for (int dy = 0; dy < 3; ++dy)
#pragma unroll
    for (int dx = 0; dx < 3; ++dx) n1[dy * 3 + dx] = kc_jacobi_zero(pf[(dy - 1) * S + (dx - 1)], st.c);
  const double au = kc_sum9(st, n1[0], n1[1], n1[2], n1[3], n1[4], n1[5], n1[6], n1[7], n1[8]);
  return kc_jacobi_pt(n1[4], pf[0], au, st.c);
}
__device__ __forceinline__ void bot_j2z(double* __restrict__ u, const double* __restrict__ f, const BotLv& L,
                                        const St9& st, int tid, int nth, const BotPush& ps) {
  const int m = L.m, S = L.S;
  if (!L.rb4) {
    for (int i = tid; i < L.nitem1; i += nth) {
      const int y = bot_div(i, L.inv), x = i - y * m;
      ps.put(u, S, y, x, bot_j2z_pt(f + y * S + x, S, st));
    }
    return;
  }
  // 2-row items (several items per thread): the u1 = 0 + c f values of rows
  // y0-1 .. y0+2 are shared by both outputs (the same rounded product
  // wherever used), and the two chains run side by side
  const int n2 = m * ((L.rows + 1) >> 1);
  for (int it = tid; it < n2; it += nth) {
    const int rb = bot_div(it, L.inv), x = it - rb * m, y0 = 2 * rb;
    const double* pf = f + y0 * S + x;
    if (y0 + 2 <= L.rows) {
      double n1[4][3];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) n1[k][dx] = kc_jacobi_zero(pf[(k - 1) * S + dx - 1], st.c);
      const double a0 = kc_sum9(st, n1[0][0], n1[0][1], n1[0][2], n1[1][0], n1[1][1], n1[1][2], n1[2][0], n1[2][1],
                                n1[2][2]);
      const double a1 = kc_sum9(st, n1[1][0], n1[1][1], n1[1][2], n1[2][0], n1[2][1], n1[2][2], n1[3][0], n1[3][1],
                                n1[3][2]);
      const double o0 = kc_jacobi_pt(n1[1][1], pf[0], a0, st.c), o1 = kc_jacobi_pt(n1[2][1], pf[S], a1, st.c);
      ps.put(u, S, y0, x, o0);
      ps.put(u, S, y0 + 1, x, o1);
    } else {
      ps.put(u, S, y0, x, bot_j2z_pt(pf, S, st));
    }
  }
}

// fc = FW(r) on the crows x mc coarse block of this CTA (fc: its row 0);
// with cc the child is the 1x1 coarsest and its solve f/center is folded in
// (coarsest_solve, cycle.py:182-190)
__device__ __forceinline__ void bot_restrict(const double* __restrict__ r, const BotLv& L, double* __restrict__ fc,
                                             int mc, int SC, double* __restrict__ vc, double ccenter, bool cc,
                                             int tid, int nth, const BotPush& ps) {
  const int S = L.S;
  const int n = L.crows * mc;
  for (int i = tid; i < n; i += nth) {
    const int q = bot_div(i, L.invc), p = i - q * mc;
    const double* rc = r + (2 * q + 1) * S + (2 * p + 1);
    const double* rs = rc - S;
    const double* rn = rc + S;
    const double fv = kc_fw(rs[-1], rs[0], rs[1], rc[-1], rc[0], rc[1], rn[-1], rn[0], rn[1]);
    ps.put(fc, SC, q, p, fv);
    if (cc) vc[0] = __ddiv_rn(fv, ccenter);
  }
}

// The same restriction into a level replicated in every CTA (the side-15
// level under frame operators): each value goes to all cs CTAs' copies.
__device__ __forceinline__ void bot_restrict_bcast(const double* __restrict__ r, const BotLv& L, double* fc, int mc,
                                                   int SC, int tid, int nth, int cs) {
  cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
  const int S = L.S;
  const int n = L.crows * mc;
  for (int i = tid; i < n; i += nth) {
    const int q = bot_div(i, L.invc), p = i - q * mc;
    const double* rc = r + (2 * q + 1) * S + (2 * p + 1);
    const double* rs = rc - S;
    const double* rn = rc + S;
    const double fv = kc_fw(rs[-1], rs[0], rs[1], rc[-1], rc[0], rc[1], rn[-1], rn[0], rn[1]);
    for (int k = 0; k < cs; ++k) *cl.map_shared_rank(fc + q * SC + p, k) = fv;
  }
}

// u += P vc (zero: u = 0 + P vc) on this CTA's rows, one coarse cell (2x2
// fine points) per item; vc points at the child row matching fine row 0 / 2
__device__ __forceinline__ void bot_prolong(double* __restrict__ u, const double* __restrict__ vc, const BotLv& L,
                                            int mc, int SC, bool zero, int tid, int nth, const BotPush& ps) {
  const int S = L.S;
  const int nc = mc + 1;
  const int n = ((L.rows + 1) >> 1) * nc;
  for (int i = tid; i < n; i += nth) {
    const int q = bot_div(i, L.invn), p = i - q * nc;
    const double c00 = vc[(q - 1) * SC + p - 1], c01 = vc[(q - 1) * SC + p];
    const double c10 = vc[q * SC + p - 1], c11 = vc[q * SC + p];
    const int y = 2 * q, x = 2 * p;
    // (even, even): fine[0::2, 0::2] = 0.25 (((c00 + c01) + c10) + c11)   (transfer.py:57)
    ps.put(u, S, y, x, DADD(zero ? 0.0 : u[y * S + x], DMUL(0.25, DADD(DADD(DADD(c00, c01), c10), c11))));
    if (p < mc)  // (even, odd): fine[0::2, 1::2] = 0.5 (c01 + c11)   (transfer.py:56)
      ps.put(u, S, y, x + 1, DADD(zero ? 0.0 : u[y * S + x + 1], DMUL(0.5, DADD(c01, c11))));
    if (y + 1 < L.rows) {
      ps.put(u, S, y + 1, x, DADD(zero ? 0.0 : u[(y + 1) * S + x], DMUL(0.5, DADD(c10, c11))));  // transfer.py:55
      if (p < mc) ps.put(u, S, y + 1, x + 1, DADD(zero ? 0.0 : u[(y + 1) * S + x + 1], c11));   // transfer.py:54
    }
  }
}

// Strip prolongation from a strip child without any exchange: the corrected
// v is formed on the CTA's own rows AND its two halo rows (-1, R) from the
// local copies of the pre-smoothed v and of the child's rows -1 .. R/2 —
// the same arithmetic the neighbour applies to those rows, so the copies stay
// bit-identical and the phase ends with a CTA barrier instead of a cluster
// barrier.  Cells q = -1 .. R/2 cover fine rows 2q (from child rows q-1, q)
// and 2q+1 (from child row q); rows outside -1 .. R or the domain are skipped.
__device__ __forceinline__ void bot_prolong_ext(double* __restrict__ u, const double* __restrict__ vc,
                                                const BotLv& L, int mc, int SC, bool zero, int tid, int nth) {
  const int S = L.S;
  const int nc = mc + 1;
  const int n = (L.R / 2 + 2) * nc;
  const int glo = -L.a, ghi = L.m - L.a;  // local rows inside the domain: [glo, ghi)
  for (int i = tid; i < n; i += nth) {
    const int qq = bot_div(i, L.invn), p = i - qq * nc;
    const int q = qq - 1;
    const double c10 = vc[q * SC + p - 1], c11 = vc[q * SC + p];
    const int y = 2 * q, x = 2 * p;
    if (q >= 0 && y <= L.R && y >= glo && y < ghi) {  // even row, transfer.py:56-57
      const double c00 = vc[(q - 1) * SC + p - 1], c01 = vc[(q - 1) * SC + p];
      double* pv = u + y * S + x;
      pv[0] = DADD(zero ? 0.0 : pv[0], DMUL(0.25, DADD(DADD(DADD(c00, c01), c10), c11)));
      if (p < mc) pv[1] = DADD(zero ? 0.0 : pv[1], DMUL(0.5, DADD(c01, c11)));
    }
    if (y + 1 <= L.R && y + 1 >= glo && y + 1 < ghi) {  // odd row, transfer.py:54-55
      double* pv = u + (y + 1) * S + x;
      pv[0] = DADD(zero ? 0.0 : pv[0], DMUL(0.5, DADD(c10, c11)));
      if (p < mc) pv[1] = DADD(zero ? 0.0 : pv[1], c11);
    }
  }
}

// Phases of the tiny frames with the side M a compile-time constant: one
// point (or coarse point / cell) per thread of the group (M*M <= its
// threads), index math folded, no item loop.  Per-point arithmetic is that
// of bot_stencil / bot_j2z / bot_restrict / bot_prolong.
template <int M>
__device__ __forceinline__ void bt_stencil(bool jac, bool zero, const double* __restrict__ u, double* __restrict__ o,
                                           const double* __restrict__ f, const St9& st, int tid) {
  constexpr int S = M + 2;
  if (tid >= M * M) return;
  const int y = tid / M, i = y * S + (tid - y * M);
  if (jac && zero) {
    o[i] = kc_jacobi_zero(f[i], st.c);
    return;
  }
  const double* p = u + i;
  const double au = kc_sum9(st, p[-S - 1], p[-S], p[-S + 1], p[-1], p[0], p[1], p[S - 1], p[S], p[S + 1]);
  o[i] = jac ? kc_jacobi_pt(p[0], f[i], au, st.c) : DSUB(f[i], au);
}
template <int M>
__device__ __forceinline__ void bt_j2z(double* __restrict__ u, const double* __restrict__ f, const St9& st, int tid) {
  constexpr int S = M + 2;
  if (tid >= M * M) return;
  const int y = tid / M, i = y * S + (tid - y * M);
  u[i] = bot_j2z_pt(f + i, S, st);
}
template <int M>
__device__ __forceinline__ void bt_restrict(const double* __restrict__ r, double* __restrict__ fc,
                                            double* __restrict__ vc, double ccenter, bool cc, int tid) {
  constexpr int S = M + 2, MC = (M - 1) / 2, SC = MC + 2;
  if (tid >= MC * MC) return;
  const int q = tid / MC, p = tid - q * MC;
  const double* rc = r + (2 * q + 1) * S + (2 * p + 1);
  const double* rs = rc - S;
  const double* rn = rc + S;
  const double fv = kc_fw(rs[-1], rs[0], rs[1], rc[-1], rc[0], rc[1], rn[-1], rn[0], rn[1]);
  fc[q * SC + p] = fv;
  if (cc) vc[0] = __ddiv_rn(fv, ccenter);
}
template <int M>
__device__ __forceinline__ void bt_prolong(double* __restrict__ u, const double* __restrict__ vc, bool zero, int tid) {
  constexpr int S = M + 2, MC = (M - 1) / 2, SC = MC + 2, NC = MC + 1;
  if (tid >= NC * NC) return;
  const int q = tid / NC, p = tid - q * NC;
  const double c00 = vc[(q - 1) * SC + p - 1], c01 = vc[(q - 1) * SC + p];
  const double c10 = vc[q * SC + p - 1], c11 = vc[q * SC + p];
  double* pu = u + (2 * q) * S + 2 * p;
  // (even, even): fine[0::2, 0::2] = 0.25 (((c00 + c01) + c10) + c11)   (transfer.py:57)
  pu[0] = DADD(zero ? 0.0 : pu[0], DMUL(0.25, DADD(DADD(DADD(c00, c01), c10), c11)));
  if (p < MC) pu[1] = DADD(zero ? 0.0 : pu[1], DMUL(0.5, DADD(c01, c11)));  // transfer.py:56
  if (q < MC) {
    pu[S] = DADD(zero ? 0.0 : pu[S], DMUL(0.5, DADD(c10, c11)));        // transfer.py:55
    if (p < MC) pu[S + 1] = DADD(zero ? 0.0 : pu[S + 1], c11);          // transfer.py:54
  }
}

// PH_TINY: whole kappa_cycle frames on sides <= KC_BOT_TINY_M (15, 7, 3 with
// the 1x1 folded into the 3x3 leaf), one named barrier / __syncwarp per
// phase, no descriptor decode.  Follows BotBuilder::rec with J2Z on, so the
// host's dry replay of the same rules knows the buffer each level ends in.
struct BotTiny {
  double* sm;
  const BotLv* lv;
  const St9* tab;
  int nu1, nu2, tid, nth;  // 32: warp 0 (__syncwarp); 64: warps 0-1 (barrier 2); 256: warps 0-7 (barrier 1)
  __device__ __forceinline__ void sync() const {
    if (nth == 32) __syncwarp();
    else if (nth == 64) asm volatile("bar.sync 2, 64;" ::: "memory");
    else asm volatile("bar.sync 1, 256;" ::: "memory");
    bot_jitter();
  }
  __device__ __forceinline__ double* buf(const BotLv& L, int b) const { return sm + (b ? L.vo1 : L.vo0); }
  template <int M>
  __device__ __forceinline__ void relax(const BotLv& L, const St9& st, int count, int& cur, int& vz) const {
    int i = 0;
    const double* f = sm + L.fo;
    if (count >= 2 && vz) {
      bt_j2z<M>(buf(L, cur), f, st, tid);
      sync();
      vz = 0;
      i = 2;
    }
    for (; i < count; ++i) {
      bt_stencil<M>(true, vz, buf(L, cur), buf(L, cur ^ 1), f, st, tid);
      sync();
      vz = 0;
      cur ^= 1;
    }
  }
  // pre-smooth + residual + restriction of level d into d+1
  template <int M>
  __device__ __forceinline__ void down(int d, const BotLv& L, const St9& st, int& cur, int& vz, bool cc) const {
    relax<M>(L, st, nu1, cur, vz);
    const double* f = sm + L.fo;
    if (!vz) {
      bt_stencil<M>(false, false, buf(L, cur), buf(L, cur ^ 1), f, st, tid);
      sync();
    }
    const BotLv C = lv[d + 1];
    bt_restrict<M>(vz ? f : buf(L, cur ^ 1), sm + C.fo, sm + C.vo0, tab[d + 1].center, cc, tid);
    sync();
  }
  // prolongation of child buffer cb + post-smoothing
  template <int M>
  __device__ __forceinline__ void up(int d, const BotLv& L, const St9& st, int& cur, int& vz, int cb) const {
    const BotLv C = lv[d + 1];
    bt_prolong<M>(buf(L, cur), buf(C, cb), vz, tid);
    sync();
    vz = 0;
    relax<M>(L, st, nu2, cur, vz);
  }
  // a 3x3 frame whose child is the coarsest (both coarsest calls folded)
  __device__ __forceinline__ void leaf(int d, int& cur, int& vz) const {
    const BotLv L = lv[d];
    const St9 st = tab[d];
    down<3>(d, L, st, cur, vz, true);
    up<3>(d, L, st, cur, vz, 0);
  }
  // side 7 (on warps 0-1: one point per thread): children are side-3 leaves
  // on warp 0 (kappa only sets how many); slot passes their final buffer
  __device__ __forceinline__ void frame7(int d, int kap, int& cur, int& vz, int* slot) const {
    const BotLv L = lv[d];
    const St9 st = tab[d];
    down<7>(d, L, st, cur, vz, false);
    int cc = 0;
    if (tid < 32) {
      const BotTiny w{sm, lv, tab, nu1, nu2, tid, 32};
      int cz = 1;
      w.leaf(d + 1, cc, cz);
      if (kap > 1) w.leaf(d + 1, cc, cz);
      if (nth > 32 && tid == 0) *slot = cc;
    }
    if (nth > 32) {
      sync();
      cc = *slot;
    }
    up<7>(d, L, st, cur, vz, cc);
  }
  // side 15 on warps 0-7; its side-7 children (kappa, kappa - 1;
  // cycle.py:215-218) on warps 0-1 while warps 2-7 wait at the named barrier
  // child_buf[0]: the side-15 frame's child buffer, child_buf[1]: the side-7 frames'
  __device__ void frame(int d, int kap, int nlev, int& cur, int& vz, int* child_buf) const {
    if (d + 2 == nlev) {
      leaf(d, cur, vz);
      return;
    }
    if (d + 3 == nlev) {
      frame7(d, kap, cur, vz, child_buf + 1);
      return;
    }
    const BotLv L = lv[d];
    const St9 st = tab[d];
    down<15>(d, L, st, cur, vz, false);
    if (tid < 64) {
      const BotTiny w{sm, lv, tab, nu1, nu2, tid, 64};
      int cc = 0, cz = 1;
      w.frame7(d + 1, kap, cc, cz, child_buf + 1);
      if (kap > 1) w.frame7(d + 1, kap - 1, cc, cz, child_buf + 1);
      if (tid == 0) child_buf[0] = cc;
    }
    sync();
    up<15>(d, L, st, cur, vz, child_buf[0]);
  }
};

#ifndef KC_MV_TWO
#define KC_MV_TWO 1
#endif
#ifndef KC_MV_ASYNC
#define KC_MV_ASYNC 1
#endif
#ifndef KC_RB_ASYNC  // the 63^2 -> 31^2 restriction broadcast of the deep frames as st.async
#define KC_RB_ASYNC 1
#endif
// the st.async phases as a runtime switch (BotParams::async) in the jitter
// builds only, where tests/test_gpu_jitter.py runs both schemes under
// perturbation; the production builds compile the st.async path alone (the
// switch cost 0.5 % per cycle there)
#ifdef KC_BOT_JITTER
#define KC_ASYNC_ON(bp, bit) ((((bp)->async) >> (bit)) & 1)
#else
#define KC_ASYNC_ON(bp, bit) true
#endif
#ifndef KC_XB_ASYNC  // the deep frames' halo exchanges (v rows) as st.async: measured no
#define KC_XB_ASYNC 0     // faster in the FMA build, 1.4 % slower per cycle in the exact one
#endif
__device__ __forceinline__ unsigned bot_sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned bot_mapa(unsigned a, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// One frame operator phase on every CTA of the cluster: this CTA's rows
// i in [rank * R, rank * R + R) of v' = A_k v + B_k f (the A part skipped on
// a zero guess), inputs gathered from CTA 0's side-15 level, outputs stored
// into CTA 0's other v buffer (so no CTA overwrites an input another CTA may
// still read); the caller ends the phase with a cluster barrier.
// (bb, ba: the blocks applied to f and to v; bb = -1 selects B_kap / A_kap)
__device__ __forceinline__ void bot_mv_frame(double* sm, const BotParams& bp, const BotLv& L, int src, int ob,
                                             bool zero, int kap, int rank, int cs, int bb = -1, int ba = -1,
                                             unsigned long long* mvb = nullptr) {
  cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
  const int R = bp.mv_rows;
  asm volatile("cp.async.wait_all;" ::: "memory");  // the blocks (prologue copies)
  bot_bar();
  KC_BOT_SUB(14);
  // this CTA's row slice of the blocks: in shared memory (resident), else
  // straight from global memory (2.4 MB for all six blocks: L2-resident)
  if (bb < 0) {
    bb = (kap - 1) * 2 + 1;
    ba = (kap - 1) * 2;
  }
  if (ba < 0) ba = bb;  // a pair operator on a zero guess: A is never read
  const int i0 = rank * R;
  const double* vin = sm + (src ? L.vo1 : L.vo0);  // this CTA's replica
  const double* fin = sm + L.fo;
  double* xv = sm + bp.mv_xin;  // inputs packed row-major: v (225), f (225)
  double* xf = xv + KC_MV_N;
  for (int i = threadIdx.x; i < KC_MV_N; i += KC_BOT_THREADS) {
    const int y = i / KC_MV_M, o = y * L.S + (i - y * KC_MV_M);
    xf[i] = fin[o];
    if (!zero) xv[i] = vin[o];
  }
  if (mvb && threadIdx.x == 0)  // this CTA's replica receives all KC_MV_N outputs of the phase
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bot_sa(mvb)), "r"(KC_MV_N * 8)
                 : "memory");
  bot_bar();
  KC_BOT_SUB(15);
  double* out = sm + (ob ? L.vo1 : L.vo0);
  // lane l's row value into CTA l's replica: a DSMEM store, or (mvb) an
  // st.async completing its bytes on CTA l's mbarrier
  auto put = [&](double* p, int l, double v) {
    if (!mvb) {
      *cl.map_shared_rank(p, l) = v;
      return;
    }
    const unsigned ra = bot_mapa(bot_sa(p), l), rb = bot_mapa(bot_sa(mvb), l);
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra), "d"(v),
                 "r"(rb)
                 : "memory");
  };
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#if KC_MV_TWO
  // two rows per warp pass (r, r + warps) with independent chains; their
  // reductions share the shuffles: one exchange splits the lanes into a row-r
  // half and a row-(r + warps) half, four more reduce within each half
  auto rows = [&](const double* B, const double* A) {
    for (int r = warp; r < R && i0 + r < KC_MV_N; r += 2 * KC_BOT_WARPS) {
      const int r2 = r + KC_BOT_WARPS;
      const bool two = r2 < R && i0 + r2 < KC_MV_N;
      const double* br = B + r * KC_MV_LD;
      const double* ar = A + r * KC_MV_LD;
      const double* br2 = B + (two ? r2 : r) * KC_MV_LD;
      const double* ar2 = A + (two ? r2 : r) * KC_MV_LD;
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
      for (int k = 0; k < (KC_MV_N + 31) / 32; ++k) {
        const int j = lane + 32 * k;
        if (j < KC_MV_N) {
          const double x = xf[j];
          a0 = fma(br[j], x, a0);
          b0 = fma(br2[j], x, b0);
          if (!zero) {
            const double y = xv[j];
            a1 = fma(ar[j], y, a1);
            b1 = fma(ar2[j], y, b1);
          }
        }
      }
      const double va = a0 + a1, vb = b0 + b1;
      const bool hi = lane >= 16;
      double acc = (hi ? vb : va) + __shfl_xor_sync(0xffffffffu, hi ? va : vb, 16);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      // lanes 0-15: row r, lanes 16-31: row r2; lane k & 15 stores into CTA k's replica
      const int i = i0 + (hi ? r2 : r), y = i / KC_MV_M, x = i - y * KC_MV_M;
      if ((lane & 15) < cs && (!hi || two)) put(out + y * L.S + x, lane & 15, acc);
    }
  };
#else
  auto rows = [&](const double* B, const double* A) {
    for (int r = warp; r < R && i0 + r < KC_MV_N; r += KC_BOT_WARPS) {
      const double* br = B + r * KC_MV_LD;
      const double* ar = A + r * KC_MV_LD;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;  // independent chains
#pragma unroll
      for (int k = 0; k < (KC_MV_N + 31) / 32; ++k) {
        const int j = lane + 32 * k;
        if (j < KC_MV_N) {
          if (k & 1) a1 = fma(br[j], xf[j], a1);
          else a0 = fma(br[j], xf[j], a0);
          if (!zero) {
            if (k & 1) a3 = fma(ar[j], xv[j], a3);
            else a2 = fma(ar[j], xv[j], a2);
          }
        }
      }
      double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      // every lane holds the row's value: lane k stores it into CTA k's replica
      const int i = i0 + r, y = i / KC_MV_M, x = i - y * KC_MV_M;
      if (lane < cs) put(out + y * L.S + x, lane, acc);
    }
  };
#endif
  // shared-memory loads where the blocks are resident (a pointer that may
  // be either would make every load a generic one)
  const int sb = bp.mv_slot[bb], sa = bp.mv_slot[ba];
  if (sb >= 0 && (zero || sa >= 0))
    rows(sm + bp.mv_off + sb * R * KC_MV_LD, sm + bp.mv_off + (zero ? sb : sa) * R * KC_MV_LD);
  else
    rows(bp.mv_mats + ((size_t)bb * KC_MV_N + i0) * KC_MV_LD, bp.mv_mats + ((size_t)ba * KC_MV_N + i0) * KC_MV_LD);
  KC_BOT_SUB(16);
}
// the end of an st.async frame-operator phase (bot_mv_frame with mvb): every
// thread waits until all KC_MV_N outputs have landed in this CTA's replica
// (phase parity ph of this mbarrier).  No cluster barrier: a CTA that passes
// has every CTA's outputs, so every CTA is past its input reads; the next
// phase writes the other buffer, into the other mbarrier.
__device__ __forceinline__ void bot_mv_wait(unsigned long long* mvb, unsigned ph) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W%=;\n}" ::"r"(
          bot_sa(mvb)),
      "r"(ph)
      : "memory");
  bot_jitter();
}

// PH_FRAME31: a whole kappa_cycle frame on the replicated side-31 level --
// its sweeps, residual, restriction, the side-15 frames below it (frame
// operators, or BotTiny on warps 0-7) and the prolongation -- with the side
// a compile-time constant: no descriptor decode, folded index math, CTA
// barriers only (every CTA works on its own copy; the frame operators add
// their cluster barrier).  Follows BotBuilder::rec_plain and the frame-
// operator bookkeeping (mv_last / mv_sync), which the host replays dry.
struct BotFrame31 {
  static constexpr int M = 31, S = M + 2, MC = 15, SC = MC + 2;
  double* sm;
  const BotLv* lv;
  const St9* tab;
  const BotParams* bp;
  int tid, rank, cs, nlev;
  int* slot;      // shared int: a BotTiny frame's final buffer for the other warps
  int* tiny_child;
  int mv_last;    // buffer the previous frame operator wrote (-1: none)
  bool mv_sync;   // an interpreter frame ran since the last frame operator
  unsigned long long* mvbar;  // two mbarriers for the st.async frame-operator phases (KC_MV_ASYNC)
  int mv_n;                   // st.async phases so far this launch (the same count on every CTA)
  int rb_n;                   // st.async restriction broadcasts into the 31^2 replicas so far (KC_RB_ASYNC)
  int xb_n;                   // st.async deep-halo exchanges so far (KC_XB_ASYNC)
  // one frame-operator phase and its completion: bot_mv_frame, then the
  // cluster barrier, or (KC_MV_ASYNC) the wait on this CTA's mbarrier
  __device__ __forceinline__ void mv(const BotLv& L, int src, int ob, bool zero, int kap, int bb = -1) {
    if (KC_MV_ASYNC && cs > 1 && KC_ASYNC_ON(bp, 0)) {
      unsigned long long* b = mvbar + (mv_n & 1);
      bot_mv_frame(sm, *bp, L, src, ob, zero, kap, rank, cs, bb, -1, b);
      bot_mv_wait(b, (mv_n >> 1) & 1);
      ++mv_n;
    } else {
      bot_mv_frame(sm, *bp, L, src, ob, zero, kap, rank, cs, bb);
      clu_sync();
    }
  }
  __device__ __forceinline__ double* buf(const BotLv& L, int b) const { return sm + (b ? L.vo1 : L.vo0); }
  __device__ __forceinline__ void stencil(bool jac, bool zero, const double* u, double* o, const double* f,
                                          const St9& st) const {
    const BotPush ps{nullptr, nullptr, 0, 1 << 30};
    bot_stencil<4>(jac, zero, u, o, f, M, M, S, 1.0f / (float)M, st, tid, KC_BOT_THREADS, M * ((M + 3) / 4), ps);
  }
  __device__ __forceinline__ void j2z(double* u, const double* f, const St9& st) const {
    // 2-row items sharing their u1 = 0 + c f values (bot_j2z)
    for (int it = tid; it < M * ((M + 1) / 2); it += KC_BOT_THREADS) {
      const int rb = it / M, x = it - rb * M, y0 = 2 * rb;
      const double* pf = f + y0 * S + x;
      if (y0 + 2 <= M) {
        double n1[4][3];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) n1[k][dx] = kc_jacobi_zero(pf[(k - 1) * S + dx - 1], st.c);
        const double a0 = kc_sum9(st, n1[0][0], n1[0][1], n1[0][2], n1[1][0], n1[1][1], n1[1][2], n1[2][0],
                                  n1[2][1], n1[2][2]);
        const double a1 = kc_sum9(st, n1[1][0], n1[1][1], n1[1][2], n1[2][0], n1[2][1], n1[2][2], n1[3][0],
                                  n1[3][1], n1[3][2]);
        u[y0 * S + x] = kc_jacobi_pt(n1[1][1], pf[0], a0, st.c);
        u[(y0 + 1) * S + x] = kc_jacobi_pt(n1[2][1], pf[S], a1, st.c);
      } else {
        u[y0 * S + x] = bot_j2z_pt(pf, S, st);
      }
    }
  }
  __device__ __forceinline__ void relax(const BotLv& L, const St9& st, int count, int& cur, int& vz) const {
    int i = 0;
    const double* f = sm + L.fo;
    if (count >= 2 && vz) {
      j2z(buf(L, cur), f, st);
      bot_bar();
      vz = 0;
      i = 2;
    }
    for (; i < count; ++i) {
      stencil(true, vz, buf(L, cur), buf(L, cur ^ 1), f, st);
      bot_bar();
      vz = 0;
      cur ^= 1;
    }
  }
  // the side-15 frame below (frame operator or BotTiny), with its buffer
  __device__ __forceinline__ void frame15(int d, int kap, int& c, int& z) {
    const int k3 = kap < 3 ? kap : 3;
    const int need = (1 << ((k3 - 1) * 2 + 1)) | (z ? 0 : (1 << ((k3 - 1) * 2)));
    if (KC_FAST && (bp->mv_avail & need) == need) {  // frame operators exist in the FMA build only
      if (mv_sync) clu_sync();
      mv_sync = false;
      const int ob = z ? (mv_last >= 0 ? mv_last ^ 1 : c ^ 1) : c ^ 1;
      mv(lv[d], c, ob, z, k3);
      mv_last = ob;
      c = ob;
      z = 0;
      return;
    }
    if (bp->mv_avail) mv_sync = true;
    if (tid < 256) {
      const BotTiny t{sm, lv, tab, bp->nu1, bp->nu2, tid, 256};
      t.frame(d, kap, nlev, c, z, tiny_child);
      if (tid == 0) *slot = c;
    }
    bot_bar();
    c = *slot;
    z = 0;
  }
  __device__ __forceinline__ void frame(int d, int kap, int& cur, int& vz) {
    const BotLv L = lv[d], C = lv[d + 1];
    const St9 st = tab[d];
    const int nu1 = bp->nu1, nu2 = bp->nu2;
    KC_BOT_SUB(7);
    relax(L, st, nu1, cur, vz);
    KC_BOT_SUB(8);
    const double* f = sm + L.fo;
    if (!vz) {
      stencil(false, false, buf(L, cur), buf(L, cur ^ 1), f, st);
      bot_bar();
    }
    KC_BOT_SUB(9);
    {  // full weighting into the child's f (transfer.py:78-83)
      const double* r = vz ? f : buf(L, cur ^ 1);
      double* fc = sm + C.fo;
      for (int i = tid; i < MC * MC; i += KC_BOT_THREADS) {
        const int q = i / MC, p = i - q * MC;
        const double* rc = r + (2 * q + 1) * S + (2 * p + 1);
        const double* rs = rc - S;
        const double* rn = rc + S;
        fc[q * SC + p] = kc_fw(rs[-1], rs[0], rs[1], rc[-1], rc[0], rc[1], rn[-1], rn[0], rn[1]);
      }
      bot_bar();
    }
    KC_BOT_SUB(10);
    int c = 0, z = 1;  // the child's zero guess (cycle.py:214)
    if (KC_FAST && kap > 1 && ((bp->mv_avail >> kc_mv_pair(kap)) & 1)) {
      // both frames (kap, kap - 1) from the zero guess as one operator
      if (mv_sync) clu_sync();
      mv_sync = false;
      const int ob = mv_last >= 0 ? mv_last ^ 1 : c ^ 1;
      mv(lv[d + 1], c, ob, true, kap, kc_mv_pair(kap));
      mv_last = ob;
      c = ob;
      z = 0;
    } else {
      frame15(d + 1, kap, c, z);
      if (kap > 1) frame15(d + 1, kap - 1, c, z);
    }
    KC_BOT_SUB(11);
    {  // u += P vc, one coarse cell (2x2 fine points) per item (transfer.py:50-58)
      double* u = buf(L, cur);
      const double* vc = buf(C, c);
      constexpr int NC = MC + 1;
      for (int i = tid; i < NC * NC; i += KC_BOT_THREADS) {
        const int q = i / NC, p = i - q * NC;
        const double c00 = vc[(q - 1) * SC + p - 1], c01 = vc[(q - 1) * SC + p];
        const double c10 = vc[q * SC + p - 1], c11 = vc[q * SC + p];
        double* pu = u + (2 * q) * S + 2 * p;
        pu[0] = DADD(vz ? 0.0 : pu[0], DMUL(0.25, DADD(DADD(DADD(c00, c01), c10), c11)));
        if (p < MC) pu[1] = DADD(vz ? 0.0 : pu[1], DMUL(0.5, DADD(c01, c11)));
        if (q < MC) {
          pu[S] = DADD(vz ? 0.0 : pu[S], DMUL(0.5, DADD(c10, c11)));
          if (p < MC) pu[S + 1] = DADD(vz ? 0.0 : pu[S + 1], c11);
        }
      }
      bot_bar();
    }
    KC_BOT_SUB(12);
    vz = 0;
    relax(L, st, nu2, cur, vz);
    KC_BOT_SUB(13);
  }
};

// PH_FRAME63: the pair of calls (kappa, kappa - 1) on the side-63 strip
// level (cycle.py:215-218) with DEEP halos.  Each CTA owns R = 4 rows and
// keeps KC_DEEP_HB = 4 halo rows each side, and computes every stage of a
// call on as many halo rows as the later stages need -- redundantly, with
// CTA barriers only -- so a call needs a cluster barrier only where data
// must cross CTAs: the restriction into the replicated 31^2 level (broadcast)
// and, for the continuing call, one exchange of v's rows before its sweeps
// and one of the boundary rows after them (the parent's prolongation reads
// one halo row).  Zero-guess call: J2Z on rows -3..R+2 (f halo 4), residual
// on -1..R, restriction of the own coarse rows, the 31^2 frames (BotFrame31),
// prolongation on -3..R+2, sweeps on -2..R+1 and -1..R.  Continuing call:
// exchange v (depth 4), sweeps on -3..R+2 and -2..R+1, residual, restriction,
// frames, prolongation on -2..R+1, sweeps on -1..R and 0..R-1, exchange of
// the boundary rows.  Rows outside the domain are never written (they stay
// the zero Dirichlet ghosts).  Same per-point arithmetic and buffer rules as
// BotBuilder::rec_plain (nu1 = nu2 = 2): bit-identical to the strip phases.
//
// PH_FRAME127 (a whole launch from a zero guess on the 127^2 entry level):
// the same scheme one level up -- 127^2 strips of R = 8 rows with deep halos
// too (the entry load brings 4 halo rows of f), its pair of calls around the
// 63^2 pairs.  Its restriction writes the child's strip rows AND pushes them
// into both neighbours' deep halos (4 rows = a whole 63^2 strip), so the
// 63^2 calls start without an exchange; the last 63^2 call of each pair
// pushes 2 boundary rows (the 127^2 prolongation of rows -2..R+1 reads child
// rows -2..R/2), and the 127^2 post pass keeps only its own rows valid (the
// next call exchanges depth 4, the last one is written back).  Cluster
// barriers per 127^2 call: 1 (zero guess) or 3, against 6-7 strip phases.
struct BotDeep {
  static constexpr int HB = KC_DEEP_HB;
  double* sm;
  const BotLv* lv;
  const St9* tab;
  BotFrame31* f31;
  int tid, rank, cs;
  __device__ __forceinline__ double* buf(const BotLv& L, int b) const { return sm + (b ? L.vo1 : L.vo0); }
  // items (y, x) of rows lo..hi clipped to the domain (local row y = global a + y)
  template <int M, class Fn>
  __device__ __forceinline__ void rows_do(int a, int lo, int hi, Fn fn) const {
    lo = max(lo, -a);
    hi = min(hi, M - 1 - a);
    const int n = (hi - lo + 1) * M;
    for (int i = tid; i < n; i += KC_BOT_THREADS) {
      const int yy = i / M;
      fn(lo + yy, i - yy * M);
    }
  }
  // a Jacobi sweep (JAC) or the residual on rows lo..hi (clipped): items of
  // two rows sharing their loads (12 instead of 18 per pair), the per-point
  // arithmetic of kc_apply9 / kc_jacobi_pt
  template <int M, bool JAC>
  __device__ __forceinline__ void stencil2(int a, int lo, int hi, const double* __restrict__ u, double* __restrict__ o,
                                           const double* __restrict__ f, const St9& st) const {
    constexpr int S = M + 2;
    lo = max(lo, -a);
    hi = min(hi, M - 1 - a);
    const int n = ((hi - lo + 2) >> 1) * M;
    for (int it = tid; it < n; it += KC_BOT_THREADS) {
      const int yy = it / M, x = it - yy * M, y = lo + 2 * yy;
      const bool two = y + 1 <= hi;
      const int i = y * S + x;
      const double* q = u + i;
      double r[4][3];
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) r[k][dx] = q[(k - 1) * S + dx - 1];
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) r[3][dx] = two ? q[2 * S + dx - 1] : 0.0;
      const double a0 = kc_sum9(st, r[0][0], r[0][1], r[0][2], r[1][0], r[1][1], r[1][2], r[2][0], r[2][1], r[2][2]);
      const double a1 = kc_sum9(st, r[1][0], r[1][1], r[1][2], r[2][0], r[2][1], r[2][2], r[3][0], r[3][1], r[3][2]);
      o[i] = JAC ? kc_jacobi_pt(r[1][1], f[i], a0, st.c) : DSUB(f[i], a0);
      if (two) o[i + S] = JAC ? kc_jacobi_pt(r[2][1], f[i + S], a1, st.c) : DSUB(f[i + S], a1);
    }
  }
  // u += P vc on rows lo..hi (clipped) by coarse cells: cell (q, p) holds the
  // fine points (2q|2q+1, 2p|2p+1) of global rows and reads the four coarse
  // values they share (cp(q, p): coarse row q by its global index) -- no
  // divergence on the column parity, 4 loads per 4 points; the arithmetic of
  // kc_prolong_val (transfer.py:54-57)
  template <int M, class CP>
  __device__ __forceinline__ void prolong_cells(int a, int lo, int hi, double* __restrict__ u, CP cp) const {
    constexpr int S = M + 2, NC = (M + 1) / 2;
    lo = max(lo, -a);
    hi = min(hi, M - 1 - a);
    const int q0 = (a + lo) >> 1, q1 = (a + hi) >> 1;
    const int n = (q1 - q0 + 1) * NC;
    for (int it = tid; it < n; it += KC_BOT_THREADS) {
      const int qq = it / NC, pc = it - qq * NC, q = q0 + qq;
      const double c00 = cp(q - 1, pc - 1), c01 = cp(q - 1, pc), c10 = cp(q, pc - 1), c11 = cp(q, pc);
      const int ly = 2 * q - a, x = 2 * pc;
      const bool xo = x + 1 < M;
      if (ly >= lo && ly <= hi) {  // fine row 2q
        double* pu = u + ly * S + x;
        pu[0] = DADD(pu[0], DMUL(0.25, DADD(DADD(DADD(c00, c01), c10), c11)));
        if (xo) pu[1] = DADD(pu[1], DMUL(0.5, DADD(c01, c11)));
      }
      if (ly + 1 >= lo && ly + 1 <= hi) {  // fine row 2q + 1
        double* pu = u + (ly + 1) * S + x;
        pu[0] = DADD(pu[0], DMUL(0.5, DADD(c10, c11)));
        if (xo) pu[1] = DADD(pu[1], c11);
      }
    }
  }
  // J2Z (two sweeps from the zero guess, bot_j2z_pt) on two-row items: the
  // u1 = 0 + c f values of rows y-1 .. y+2 shared by both outputs
  template <int M>
  __device__ __forceinline__ void j2z2(int a, int lo, int hi, double* __restrict__ u, const double* __restrict__ f,
                                       const St9& st) const {
    constexpr int S = M + 2;
    lo = max(lo, -a);
    hi = min(hi, M - 1 - a);
    const int n = ((hi - lo + 2) >> 1) * M;
    for (int it = tid; it < n; it += KC_BOT_THREADS) {
      const int yy = it / M, x = it - yy * M, y = lo + 2 * yy;
      const bool two = y + 1 <= hi;
      const int i = y * S + x;
      const double* pf = f + i;
      double n1[4][3];
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) n1[k][dx] = kc_jacobi_zero(pf[(k - 1) * S + dx - 1], st.c);
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) n1[3][dx] = two ? kc_jacobi_zero(pf[2 * S + dx - 1], st.c) : 0.0;
      const double a0 =
          kc_sum9(st, n1[0][0], n1[0][1], n1[0][2], n1[1][0], n1[1][1], n1[1][2], n1[2][0], n1[2][1], n1[2][2]);
      const double a1 =
          kc_sum9(st, n1[1][0], n1[1][1], n1[1][2], n1[2][0], n1[2][1], n1[2][2], n1[3][0], n1[3][1], n1[3][2]);
      u[i] = kc_jacobi_pt(n1[1][1], pf[0], a0, st.c);
      if (two) u[i + S] = kc_jacobi_pt(n1[2][1], pf[S], a1, st.c);
    }
  }
  // own rows ylo..yhi into the neighbours' halo rows: rows y < HB to the
  // upper one (its row R + y), rows y >= R - HB to the lower one (row y - R)
  template <int M>
  __device__ __forceinline__ void push_rows(double* u, int a, int ylo, int yhi) const {
    constexpr int R = (M + 1) / 16, S = M + 2;
    if (KC_XB_ASYNC) {  // st.async completing on the neighbour's exchange mbarrier
      const unsigned ub = bot_sa(u), bb = bot_sa(f31->mvbar + 3);
      const bool hu = rank > 0, hd = rank + 1 < cs;
      const unsigned bu = hu ? bot_mapa(bb, rank - 1) : 0u, bd = hd ? bot_mapa(bb, rank + 1) : 0u;
      rows_do<M>(a, ylo, yhi, [&](int y, int x) {
        const double v = u[y * S + x];
        if (hu && y < HB)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(
                           bot_mapa(ub + 8u * (unsigned)((R + y) * S + x), rank - 1)),
                       "d"(v), "r"(bu)
                       : "memory");
        if (hd && y >= R - HB)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(
                           bot_mapa(ub + 8u * (unsigned)((y - R) * S + x), rank + 1)),
                       "d"(v), "r"(bd)
                       : "memory");
      });
      return;
    }
    cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
    double* up = rank > 0 ? cl.map_shared_rank(u, rank - 1) + R * S : nullptr;
    double* dn = rank + 1 < cs ? cl.map_shared_rank(u, rank + 1) - R * S : nullptr;
    rows_do<M>(a, ylo, yhi, [&](int y, int x) {
      const double v = u[y * S + x];
      if (up && y < HB) up[y * S + x] = v;
      if (dn && y >= R - HB) dn[y * S + x] = v;
    });
  }
  // bytes this CTA receives when every CTA runs push_rows<M>(.., ylo, yhi):
  // rows y < HB of the CTA below it, rows y >= R - HB of the one above
  template <int M>
  __device__ __forceinline__ int push_bytes(int ylo, int yhi) const {
    constexpr int R = (M + 1) / 16;
    auto cnt = [&](int s, bool to_up) {
      const int hi = min(yhi, M - 1 - s * R);
      int c = 0;
      for (int y = ylo; y <= hi; ++y) c += to_up ? (y < HB) : (y >= R - HB);
      return c;
    };
    int n = 0;
    if (rank + 1 < cs) n += cnt(rank + 1, true);
    if (rank > 0) n += cnt(rank - 1, false);
    return n * M * 8;
  }
  // a halo exchange of push_rows: the expected bytes on this CTA's exchange
  // mbarrier before the pushes, the wait after them (KC_XB_ASYNC), else the
  // cluster barrier.  Every exchange is preceded by a cluster barrier (the
  // write-after-read guard), so the next exchange's bytes cannot reach this
  // CTA before it has waited for this one: one mbarrier serves.
  __device__ __forceinline__ void xchg_begin(int bytes) const {
    if (KC_XB_ASYNC && tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bot_sa(f31->mvbar + 3)),
                   "r"(bytes)
                   : "memory");
  }
  __device__ __forceinline__ void xchg_end() const {
    if (KC_XB_ASYNC) {
      bot_mv_wait(f31->mvbar + 3, f31->xb_n & 1);
      ++f31->xb_n;
    } else {
      clu_sync();
    }
  }
  // the pre half of a call: sweeps (J2Z on a zero guess), residual,
  // restriction -- broadcast into the child's replicas (M = 63) or into the
  // child's strips with their deep halos (M = 127); returns the first row on
  // which v after the sweeps is valid (the last is R - 1 - lo)
  template <int M>
  __device__ __forceinline__ int pre(int d, int cur, bool zero) {
    constexpr int R = (M + 1) / 16, S = M + 2, MC = (M - 1) / 2, SC = MC + 2;
    const BotLv L = lv[d];
    const St9 st = tab[d];
    const int a = rank * R;
    const double* f = sm + L.fo;
    double* u = buf(L, cur);
    double* w = buf(L, cur ^ 1);
    int lo;
    if (zero) {
      j2z2<M>(a, -3, R + 2, u, f, st);
      bot_bar();
      lo = -3;
    } else {
      // v of the previous call, depth 4, into the neighbours' halo rows --
      // after a barrier: a neighbour may still be using those rows for the
      // previous call's prolongation and sweeps
      clu_sync();
      xchg_begin(push_bytes<M>(0, R - 1));
      push_rows<M>(u, a, 0, R - 1);
      xchg_end();
      stencil2<M, true>(a, -3, R + 2, u, w, f, st);
      bot_bar();
      stencil2<M, true>(a, -2, R + 1, w, u, f, st);
      bot_bar();
      lo = -2;
    }
    // residual into the other buffer, restriction of the own coarse rows
    stencil2<M, false>(a, -1, R, u, w, f, st);
    bot_bar();
    {
      cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
      const int n = L.crows * MC;
      double* fc0 = sm + lv[d + 1].fo;
      if (M == 127) {  // the child's strip (row 0 = coarse row a / 2) and its neighbours' deep halos
        constexpr int RC = R / 2;
        double* up = rank > 0 ? cl.map_shared_rank(fc0, rank - 1) + RC * SC : nullptr;
        double* dn = rank + 1 < cs ? cl.map_shared_rank(fc0, rank + 1) - RC * SC : nullptr;
        for (int i = tid; i < n; i += KC_BOT_THREADS) {
          const int q = i / MC, p = i - q * MC;
          const double* rc = w + (2 * q + 1) * S + (2 * p + 1);
          const double* rs = rc - S;
          const double* rn = rc + S;
          const double fv = kc_fw(rs[-1], rs[0], rs[1], rc[-1], rc[0], rc[1], rn[-1], rn[0], rn[1]);
          fc0[q * SC + p] = fv;
          if (up && q < HB) up[q * SC + p] = fv;
          if (dn && q >= RC - HB) dn[q * SC + p] = fv;
        }
      } else {  // every CTA's replica of the child, at this strip's first coarse row
        double* fc = fc0 + (a / 2) * SC;
        unsigned long long* rb = f31->mvbar + 2;
        const bool as = KC_RB_ASYNC && KC_ASYNC_ON(f31->bp, 1);
        if (as && tid == 0)  // this CTA's replica receives the whole MC x MC child f
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bot_sa(rb)), "r"(MC * MC * 8)
                       : "memory");
        for (int i = tid; i < n; i += KC_BOT_THREADS) {
          const int q = i / MC, p = i - q * MC;
          const double* rc = w + (2 * q + 1) * S + (2 * p + 1);
          const double* rs = rc - S;
          const double* rn = rc + S;
          const double fv = kc_fw(rs[-1], rs[0], rs[1], rc[-1], rc[0], rc[1], rn[-1], rn[0], rn[1]);
          if (as) {
            const unsigned la = bot_sa(fc + q * SC + p), lb = bot_sa(rb);
            for (int k = 0; k < cs; ++k)
              asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(
                               bot_mapa(la, k)),
                           "d"(fv), "r"(bot_mapa(lb, k))
                           : "memory");
          } else {
            for (int k = 0; k < cs; ++k) *cl.map_shared_rank(fc + q * SC + p, k) = fv;
          }
        }
        if (as) {
          // every CTA's rows landed here; no cluster barrier: between this
          // CTA's last read of the child's f and any CTA's next broadcast
          // lies a cluster barrier (the next call's v exchange, the 127^2
          // restriction or the interpreter's phases), so one mbarrier serves
          bot_mv_wait(rb, f31->rb_n & 1);
          ++f31->rb_n;
          return lo;
        }
      }
    }
    clu_sync();
    return lo;
  }
  // the post half of a 63^2 call: prolongation from the child's local
  // replica (buffer c), two sweeps; then np boundary rows to the neighbours
  // (1: the continuing call under a 127^2 interpreter parent, which reads one
  // halo row; 2: the last call of a pair under PH_FRAME127)
  __device__ __forceinline__ void post63(int d, int cur, int c, int lo, int np) {
    constexpr int M = 63, R = 4, S = M + 2, SC = 31 + 2;
    const BotLv L = lv[d];
    const St9 st = tab[d];
    const int a = rank * R, hi = R - 1 - lo;
    const double* f = sm + L.fo;
    double* u = buf(L, cur);
    double* w = buf(L, cur ^ 1);
    {
      const double* vc = buf(lv[d + 1], c);
      auto cp = [&](int q, int pc) { return vc[q * SC + pc]; };
      prolong_cells<M>(a, lo, hi, u, cp);
    }
    bot_bar();
    stencil2<M, true>(a, lo + 1, hi - 1, u, w, f, st);
    bot_bar();
    stencil2<M, true>(a, lo + 2, hi - 2, w, u, f, st);
    bot_bar();
    if (np > 0) {  // after a barrier: the neighbours' post sweeps read their halo rows
      clu_sync();
      xchg_begin(push_bytes<M>(0, np - 1) + push_bytes<M>(R - np, R - 1));
      push_rows<M>(u, a, 0, np - 1);
      push_rows<M>(u, a, R - np, R - 1);
      xchg_end();
    }
  }
  // the post half of a 127^2 call under PH_FRAME127: prolongation from the
  // child's strip (buffer c, local row 0 = coarse row a / 2) on rows
  // -2..R+1, sweeps on -1..R and 0..R-1 (own rows only: see above)
  __device__ __forceinline__ void post127(int cur, int c) {
    constexpr int M = 127, R = 8, S = M + 2, SC = 63 + 2;
    const BotLv L = lv[0];
    const St9 st = tab[0];
    const int a = rank * R;
    const double* f = sm + L.fo;
    double* u = buf(L, cur);
    double* w = buf(L, cur ^ 1);
    {
      const double* vc = buf(lv[1], c) - (a / 2) * SC;  // indexed by the global coarse row
      auto cp = [&](int q, int pc) { return vc[q * SC + pc]; };
      prolong_cells<M>(a, -2, R + 1, u, cp);
    }
    bot_bar();
    stencil2<M, true>(a, -1, R, u, w, f, st);
    bot_bar();
    stencil2<M, true>(a, 0, R - 1, w, u, f, st);
    bot_bar();
  }
  // PH_FRAME63 (top = false: the pair on level d63, v in buffer cur) or
  // PH_FRAME127 (top: the 127^2 pair from a zero guess, v in buffer cur, the
  // 63^2 level's v in buffer 0 as BotBuilder::rec_plain leaves it); one
  // inlined site of each half and of the child frame
  __device__ __forceinline__ void run(bool top, int d63, int kap, int cur) {
    const int ni = top ? (kap > 1 ? 2 : 1) : 1;
    for (int i = 0; i < ni; ++i) {
      KC_BOT_SUB(1);
      if (top) pre<127>(0, cur, i == 0);
      const int k1 = top ? kap - i : kap;
      const int cur63 = top ? 0 : cur;
      const int nj = k1 > 1 ? 2 : 1;
      for (int j = 0; j < nj; ++j) {
        const bool zero = j == 0;
        KC_BOT_SUB(2);
        const int lo = pre<63>(d63, cur63, zero);
        KC_BOT_SUB(3);
        int c = 0, z = 1;  // the child's zero guess (cycle.py:214)
        for (int jj = 0; jj < (k1 - j > 1 ? 2 : 1); ++jj) f31->frame(d63 + 1, k1 - j - jj, c, z);
        KC_BOT_SUB(4);
        post63(d63, cur63, c, lo, top ? (j == nj - 1 ? 2 : 0) : (zero ? 0 : 1));
      }
      KC_BOT_SUB(5);
      if (top) post127(cur, cur63);
      KC_BOT_SUB(6);
    }
  }
};

// The compile-time frames, out of line so that the interpreter loop of
// k_bottom does not carry their registers: PH_FRAME31 (one call on the
// replicated side-31 level) or PH_FRAME63 (the call pair on the deep-halo
// side-63 strips).  mvs: the frame-operator bookkeeping (mv_last, mv_sync,
// mv_n); mvbar: the two mbarriers of the st.async frame-operator phases.
__device__ __forceinline__ void bot_run_frame(int op, double* sm, const BotLv* lv, const St9* tab, const BotParams* bp,
                                           int d, int kap, int src, int zero, int rank, int cs, int nlev, int* slot,
                                           int* tiny_child, int* mvs, unsigned long long* mvbar) {
  BotFrame31 fr{sm, lv, tab, bp, (int)threadIdx.x, rank, cs, nlev, slot, tiny_child, mvs[0], mvs[1] != 0, mvbar, mvs[2], mvs[3], mvs[4]};
  if (op == PH_FRAME63 || op == PH_FRAME127) {
    BotDeep dp{sm, lv, tab, &fr, (int)threadIdx.x, rank, cs};
    dp.run(op == PH_FRAME127, op == PH_FRAME127 ? 1 : d, kap, src);
  } else {
    int cur = src, vz = zero;
    fr.frame(d, kap, cur, vz);
  }
  mvs[0] = fr.mv_last;
  mvs[1] = fr.mv_sync ? 1 : 0;
  mvs[2] = fr.mv_n;
  mvs[3] = fr.rb_n;
  mvs[4] = fr.xb_n;
}

// Columns of the side-15 frame operators: CTA (j, k - 1) runs BotTiny::frame
// (the bottom kernel's own frame code) with counter k on the unit input j
// (j < 225: v = e_j; else f = e_(j-225)) and stores v_out as column j of
// [A_k | B_k].  tp: the 4-level geometry of a side-15 entry.
// blockIdx.y >= 3: the pair operators (KC_MV_PAIR0 + y - 3): CTA j (< 225)
// runs the two frames a side-31 call makes, (2, 1), (3, 2) or (3, 3), from a
// zero v on f = e_j.  One call site of BotTiny::frame in this kernel: a
// second one (a separate pair kernel) changed how the frame code is inlined
// into k_bottom and slowed the exact build's cycle by 6 %.
__global__ void __launch_bounds__(256) k_tiny_mats(const BotParams tp, double* __restrict__ mats) {
  extern __shared__ double sm[];
  __shared__ St9 tab[4];
  __shared__ BotLv lv[4];
  __shared__ int child[2];
  const bool pair = blockIdx.y >= 3;
  const int j = blockIdx.x, py = blockIdx.y - 3;
  if (pair && j >= KC_MV_N) return;  // pairs take f inputs only
  const int ka = pair ? (py == 0 ? 2 : 3) : blockIdx.y + 1, kb = py == 0 ? 1 : (py == 1 ? 2 : 3);
  for (int i = threadIdx.x; i < tp.total; i += 256) sm[i] = 0.0;
  if (threadIdx.x < 4) {
    tab[threadIdx.x] = tp.st[threadIdx.x];
    lv[threadIdx.x] = tp.lv[threadIdx.x];
  }
  bot_bar();
  const BotLv L0 = lv[0];
  if (threadIdx.x == 0) {
    const int jj = j % KC_MV_N, y = jj / KC_MV_M, x = jj - y * KC_MV_M;
    sm[(j < KC_MV_N && !pair ? L0.vo0 : L0.fo) + y * L0.S + x] = 1.0;
  }
  bot_bar();
  const BotTiny t{sm, lv, tab, tp.nu1, tp.nu2, (int)threadIdx.x, 256};
  int cur = 0, vz = 0;
  for (int s = 0; s < (pair ? 2 : 1); ++s) {
    t.frame(0, s == 0 ? ka : kb, 4, cur, vz, child);
    bot_bar();
  }
  const double* o = sm + (cur ? L0.vo1 : L0.vo0);
  double* blk = mats + (size_t)(pair ? KC_MV_PAIR0 + py : (ka - 1) * 2 + (j < KC_MV_N ? 0 : 1)) * KC_MV_N * KC_MV_LD;
  for (int i = threadIdx.x; i < KC_MV_N; i += 256) {
    const int y = i / KC_MV_M, x = i - y * KC_MV_M;
    blk[(size_t)i * KC_MV_LD + j % KC_MV_N] = o[y * L0.S + x];
  }
}


__global__ void __launch_bounds__(KC_BOT_THREADS, 1) k_bottom(const BotParams bp, int m0) {
  extern __shared__ double sm[];
  __shared__ St9 tab[KC_BOT_MAXLEV];
  __shared__ BotLv lv[KC_BOT_MAXLEV];
  __shared__ unsigned sched[KC_BOT_MAXPH];
  __shared__ int tiny_child[2];
  // mbarriers: frame-operator phases (2), 63^2 -> 31^2 broadcast, deep-halo exchanges
  __shared__ alignas(8) unsigned long long mvbar[4];
  cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
  const int rank = (int)cl.block_rank(), cs = (int)cl.num_blocks();
  if ((KC_MV_ASYNC || KC_RB_ASYNC || KC_XB_ASYNC) && threadIdx.x == 0) {  // published by the prologue's cluster barrier
    for (int b = 0; b < 4; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bot_sa(&mvbar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int nlev = bp.nlev, nstrip = bp.nstrip;
  KC_BOT_MARK(0);
  // Prologue, ordered so the global latencies overlap: schedule and level
  // constants into registers, the entry level's rows as 8-byte cp.async
  // copies straight into shared memory, then zero everything those copies
  // do not cover (ghost rings, halos, coarser levels), then publish.
  constexpr int SCHED_PER_THREAD = (KC_BOT_MAXPH + KC_BOT_THREADS - 1) / KC_BOT_THREADS;
  unsigned sreg[SCHED_PER_THREAD];
#pragma unroll
  for (int k = 0; k < SCHED_PER_THREAD; ++k) {
    const int i = threadIdx.x + k * KC_BOT_THREADS;
    sreg[k] = i < bp.nsched ? __ldg(bp.sched + i) : 0u;
  }
  const int dl = threadIdx.x < nlev ? threadIdx.x : 0;
  const St9 st_d = bp.st[dl];
  const BotLv lv_d = bp.lv[dl];
  const int total = bp.total;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  auto cp8 = [](double* dst, const double* src) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src) : "memory");
  };
  auto zero = [&](int lo, int hi) {  // sm[lo, hi)
    if (lo >= hi) return;
    if ((lo & 1) && threadIdx.x == 0) sm[lo] = 0.0;
    const int l2 = (lo + 1) >> 1, h2 = hi >> 1;
    double2* z2 = reinterpret_cast<double2*>(sm);  // dynamic smem is 16-byte aligned
    for (int i = l2 + threadIdx.x; i < h2; i += KC_BOT_THREADS) z2[i] = make_double2(0.0, 0.0);
    if ((hi & 1) && hi - 1 >= lo && threadIdx.x == KC_BOT_THREADS - 1) sm[hi - 1] = 0.0;
  };
  if (bp.mv_copy) {
    // this CTA's row slice of every resident frame-operator block (constant
    // data: issued before the dependency wait, so it overlaps the previous
    // grid; completed by the cp.async.wait_all below or in bot_mv_frame)
    const int R = bp.mv_rows, i0 = rank * R;
    const int rows = min(R, KC_MV_N - i0);
    for (int b = 0; b < KC_MV_NBLK; ++b) {
      if (!((bp.mv_copy >> b) & 1) || rows <= 0) continue;
      const double* src = bp.mv_mats + ((size_t)b * KC_MV_N + i0) * KC_MV_LD;
      double* dst = sm + bp.mv_off + bp.mv_slot[b] * R * KC_MV_LD;
      for (int c = threadIdx.x; c < rows * KC_MV_LD / 2; c += KC_BOT_THREADS) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + 2 * c);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src + 2 * c) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (nstrip > 0) {
    // strip entry: own rows plus hb halo rows each side (1, or 4 with deep
    // halos on the entry level), within the rows -1 .. m0 that exist in
    // HBM (ghost rows zero), ghost columns included; level 0 is the first
    // block: v0 rows at [0, (R+2hb) S), f rows at [2 (R+2hb) S, ...)
    const int S = bp.lv[0].S, R = bp.lv[0].R, hb = bp.lv[0].hb, a = rank * R;
    const int y0 = max(a - hb, -1), y1 = min(a + R + hb - 1, m0);
    const int w0 = (y0 - a + hb) * S, w1 = (y1 - a + hb + 1) * S;  // loaded storage rows, as an offset range
    const int fbase = 2 * (R + 2 * hb) * S;
    if (bp.v_zero) zero(0, fbase + w0);
    else {
      zero(0, w0);
      zero(w1, fbase + w0);
    }
    zero(fbase + w1, total);
    // programmatic dependent launch: everything above touched only shared
    // memory, parameters and the schedule; the entry level is the previous
    // grid's output.  The successor (a column-tile post pass) may fetch its
    // level's f and v from now on: they were final before that grid ended.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    for (int y = y0 + wid; y <= y1; y += KC_BOT_WARPS) {
      const double* gfr = bp.gf + kc_idx(bp.gP, y, -1);
      const double* gvr = bp.gv + kc_idx(bp.gP, y, -1);
      const int o = (y - a + hb) * S;
      for (int c = lane; c < S; c += 32) {
        cp8(sm + fbase + o + c, gfr + c);
        if (!bp.v_zero) cp8(sm + o + c, gvr + c);
      }
    }
  } else {
    zero(0, total);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
  }
  KC_BOT_MARK(5);
#pragma unroll
  for (int k = 0; k < SCHED_PER_THREAD; ++k) {
    const int i = threadIdx.x + k * KC_BOT_THREADS;
    if (i < bp.nsched) sched[i] = sreg[k];
  }
  KC_BOT_MARK(6);
  if (threadIdx.x < nlev) {
    const int d = threadIdx.x;
    tab[d] = st_d;
    BotLv L = lv_d;
    if (d < nstrip) {  // this rank's rows of the strip level
      L.a = rank * L.R;
      L.rows = min(L.R, L.m - L.a);
      L.nitem1 = L.rows * L.m;
      L.nitem4 = L.m * ((L.rows + 3) / 4);
      L.rb4 = L.nitem1 > KC_BOT_THREADS;
      // coarse rows whose centre fine row 2q+1 lies in this CTA's rows
      L.crows = min(L.mc, (L.a + L.rows) / 2) - L.a / 2;
    }
    lv[d] = L;
  }
  if (nstrip > 0) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    KC_BOT_MARK(1);
    clu_sync();  // every CTA initialised before any halo push lands
  } else {
    bot_bar();
    KC_BOT_MARK(1);
    const int S = m0 + 2;
    double* v = sm + S + 1;
    double* f = sm + 2 * S * S + S + 1;
    for (int y = wid; y < m0; y += KC_BOT_WARPS) {
      const double* gfr = bp.gf + kc_idx(bp.gP, y, 0);
      const double* gvr = bp.gv + kc_idx(bp.gP, y, 0);
      for (int x = lane; x < m0; x += 32) {
        cp8(f + y * S + x, gfr + x);
        if (!bp.v_zero) cp8(v + y * S + x, gvr + x);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    bot_bar();
  }

  KC_BOT_MARK(2);
  const int warp = threadIdx.x >> 5;
  const int tid = threadIdx.x;
#ifdef KC_BOT_TRACE
  int tr_n = 0;
#endif
  if (nlev == 1) {  // the entry level is the coarsest (n == 1): f / center
    if (threadIdx.x == 0) sm[4] = __ddiv_rn(sm[2 * 9 + 4], tab[0].center);
  }
  // replay the schedule: strip phases run on every CTA and end with a
  // cluster barrier; the others run on CTA 0, where a warp takes part in the
  // phases of its group only and JOIN entries gather a larger group
  __shared__ int f31_slot;
  int mv_last = -1;      // frame-operator bookkeeping shared with PH_FRAME31 (BotBuilder mirrors it)
  bool mv_sync = false;
  int mv_n = 0, rb_n = 0, xb_n = 0;
  unsigned e_next = bp.nsched > 0 ? sched[0] : 0u;
  for (int k = 0; k < bp.nsched; ++k) {
    const unsigned e = e_next;
    if (k + 1 < bp.nsched) e_next = sched[k + 1];
    const int op = BD_OP(e);
    if (op == PH_CSYNC) {
      clu_sync();
      mv_sync = false;
      continue;
    }
    const bool strip = (e & BD_STRIP_BIT) != 0u;
    const int g = bot_desc_g(e);
    if (!strip && warp >= g) continue;  // replicated levels: every CTA on its copy
    if (op == PH_JOIN) {
      bot_sync(g);
      continue;
    }
    const int d = BD_D(e);
    const int src = BD_SRC(e);
    const bool zero = BD_ZERO(e);
    const BotLv L = lv[d];
    const int m = L.m, S = L.S;
    const int nth = g * 32;
    const double* f = sm + L.fo;
    double* u = sm + (src ? L.vo1 : L.vo0);
#ifdef KC_BOT_TRACE
    if (threadIdx.x == 0 && rank == 0 && tr_n < KC_BOT_TRACE) {
      kc_bot_trace[tr_n] = clock64();
      kc_bot_trace_op[tr_n] = op * 16 + d;
      kc_bot_trace_n = ++tr_n;
    }
#endif
    if (op == PH_J2Z) {
      bot_j2z(u, f, L, tab[d], tid, nth, bot_push(u, L, strip, rank, cs));
    } else if (op <= PH_RESID) {
      double* o = sm + (src ? L.vo0 : L.vo1);
      const St9 st = tab[d];
      const BotPush ps = bot_push(o, L, strip, rank, cs);
      if (L.rb4) bot_stencil<4>(op == PH_JACOBI, zero, u, o, f, m, L.rows, S, L.inv, st, tid, nth, L.nitem4, ps);
      else bot_stencil<1>(op == PH_JACOBI, zero, u, o, f, m, L.rows, S, L.inv, st, tid, nth, L.nitem1, ps);
    } else if (op == PH_RESTRICT) {  // r in buffer src, or f itself on a zero guess
      const BotLv C = lv[d + 1];
      double* fc = sm + C.fo;
      double* vc = sm + C.vo0;
      BotPush ps{nullptr, nullptr, 0, 1 << 30};
      if (strip && d + 1 >= nstrip) {  // into every CTA's replica of the first replicated level
        bot_restrict_bcast(zero ? f : u, L, fc + (L.a / 2) * C.S, C.m, C.S, tid, nth, cs);
      } else {
        if (strip) ps = bot_push(fc, C, true, rank, cs);  // strip child: halo rows to the neighbours
        bot_restrict(zero ? f : u, L, fc, C.m, C.S, vc, tab[d + 1].center, BD_CC(e), tid, nth, ps);
      }
    } else if (op == PH_PROLONG) {
      const BotLv C = lv[d + 1];
      const double* vc = sm + (BD_CBUF(e) ? C.vo1 : C.vo0);
      if (strip && d + 1 < nstrip) {  // halo rows formed locally: no exchange (CTA barrier below)
        bot_prolong_ext(u, vc, L, C.m, C.S, zero, tid, nth);
        bot_bar();
        continue;
      }
      if (strip)  // from this CTA's replica of the child, at this strip's first coarse row
        vc += (L.a / 2) * C.S;
      bot_prolong(u, vc, L, C.m, C.S, zero, tid, nth, bot_push(u, L, strip, rank, cs));
    } else if (op == PH_FRAME63 || op == PH_FRAME31 || op == PH_FRAME127) {  // every thread of every CTA
      int mvs[5] = {mv_last, mv_sync ? 1 : 0, mv_n, rb_n, xb_n};
      bot_run_frame(op, sm, lv, tab, &bp, d, BD_KAP(e), src, zero, rank, cs, nlev, &f31_slot, tiny_child, mvs, mvbar);
      mv_last = mvs[0];
      mv_sync = mvs[1] != 0;
      mv_n = mvs[2];
      rb_n = mvs[3];
      xb_n = mvs[4];
    } else if (KC_FAST && strip) {  // PH_TINY as a frame operator (all CTAs; FMA build only)
      bot_mv_frame(sm, bp, L, src, BD_CBUF(e), zero, BD_KAP(e), rank, cs);
      mv_last = BD_CBUF(e);
    } else {  // PH_TINY (every CTA: warp 0 for sides <= 7, warps 0-7 for side 15)
      if (m == KC_MV_M && bp.mv_avail) mv_sync = true;
      const BotTiny t{sm, lv, tab, bp.nu1, bp.nu2, tid, nth};
      int cur = src, vz = zero;
      t.frame(d, BD_KAP(e), nlev, cur, vz, tiny_child);
    }
#ifdef KC_BOT_TRACE
    if (threadIdx.x == 0 && rank == 0 && tr_n - 1 < KC_BOT_TRACE) kc_bot_trace_end[tr_n - 1] = clock64();
#endif
    if (strip) clu_sync();
    else bot_sync(g);
  }
  bot_bar();
  KC_BOT_MARK(3);
  {
    const BotLv L = lv[0];
    const int S = L.S;
    const double* v = sm + (bp.final_cur ? L.vo1 : L.vo0);
    for (int y = threadIdx.x >> 5; y < L.rows; y += KC_BOT_WARPS) {
      double* g = bp.gv + kc_idx(bp.gP, L.a + y, 0);
      for (int x = threadIdx.x & 31; x < m0; x += 32) g[x] = v[y * S + x];
    }
  }
  KC_BOT_MARK(4);
}
