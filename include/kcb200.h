/*
 * kcb200.h — C-ABI of the B200-native kappa-cycle multigrid engine.
 *
 * Drop-in boundary for the hot path of the reference package `kcycle`
 * (arXiv 2010.00626; /root/reference/pkg/src/kcycle).  The reference has no
 * FFI of its own: its hot path sits behind a duck-typed "state protocol"
 * consumed by kappa_cycle / run_cycle (cycle.py:204-263) plus the outer
 * drivers solve_standalone (cycle.py:303-366) and pcg_solve
 * (krylov.py:60-141).  Each entry point below replaces one method or driver of
 * that protocol; the citation names the reference symbol whose argument
 * meaning and error behaviour it keeps.  INTEGRATION.md shows the ctypes
 * binding (the only FFI mechanism available to a pure-Python reference).
 *
 * Conventions
 *   - Levels are 1-based, 1 = finest, n = coarsest (cycle.py:20).
 *   - Grid functions cross the boundary as dense row-major float64 (ny, nx)
 *     arrays of interior nodes only (mesh.py:3-7); the library stores them
 *     padded with a zero ghost ring in HBM.
 *   - Every call returns KC_OK or an error code; the code maps onto the
 *     reference's exception types (see KC_E* below).  kc_last_error() gives
 *     the message of the last failing call on that handle (thread-local
 *     message for kc_create failures, handle==NULL).
 *   - One CUDA stream per handle; a handle is not re-entrant, distinct
 *     handles may be used from distinct threads ("a solve owns its per-level
 *     state exclusively", cycle.py:18-19).
 *   - No CPU fallback: if no sm_100 device is present kc_create fails with
 *     KC_ECUDA.
 */
#ifndef KCB200_H
#define KCB200_H

#ifdef __cplusplus
extern "C" {
#endif

#define KC_ABI_VERSION 1

/* status codes */
#define KC_OK 0
#define KC_EINVAL 1     /* reference raises ValueError            */
#define KC_ESINGULAR 2  /* reference raises numpy.linalg.LinAlgError */
#define KC_ECUDA 3      /* CUDA runtime / driver failure           */
#define KC_ENOMEM 4     /* device allocation failure               */

/* enums mirrored from the reference */
#define KC_COARSEN_FULL 0        /* Coarsening.FULL_STANDARD, mesh.py:38 */
#define KC_COARSEN_SEMI_Y 1      /* Coarsening.SEMI_Y, mesh.py:39 (per-op kernels, kc_zebra.cuh) */
#define KC_SMOOTH_JACOBI 0       /* SmootherKind.DAMPED_JACOBI, smoother.py:37 */
#define KC_SMOOTH_ZEBRA_X 1      /* SmootherKind.ZEBRA_X, smoother.py:39 */
#define KC_SMOOTH_ZEBRA_Y 2      /* SmootherKind.ZEBRA_Y, smoother.py:40 */
#define KC_SMOOTH_ZEBRA_XY 3     /* SmootherKind.ZEBRA_ALTERNATING, smoother.py:41 */
#define KC_WHICH_V 0             /* GridState.v[level-1], cycle.py:155 */
#define KC_WHICH_F 1             /* GridState.f[level-1], cycle.py:156 */
#define KC_STOP_ERROR 0          /* ||v_k|| <= ||v_0||/target (cycle.py:332-347) */
#define KC_STOP_RESIDUAL 1       /* ||f-Av_k|| <= ||f-Av_0||/target (BASELINE headline) */
#define KC_STATUS_CONVERGED 0    /* cycle.py:273 */
#define KC_STATUS_DIVERGED 1     /* cycle.py:274 */
#define KC_STATUS_MAX_CYCLES 2   /* cycle.py:275 */
#define KC_STATUS_BREAKDOWN 3    /* cycle.py:276 */

typedef struct kc_handle kc_handle;

int kc_abi_version(void);

/* Arithmetic of this build: KC_ARITH_EXACT (libkcb200.so: separately rounded
 * products and sums in the reference's order, iterates bit-identical to
 * kcycle) or KC_ARITH_FAST (libkcb200_fast.so: the same expressions with FMA
 * contraction; histories within 1e-10 and identical iteration counts).  The
 * reference has no such switch; both builds export the same entry points. */
#define KC_ARITH_EXACT 0
#define KC_ARITH_FAST 1
int kc_arith_mode(void);
const char* kc_last_error(const kc_handle* h);

/* Galerkin coarse stencil R*A*P (stencil.py:129-148), bit-identical to the
 * reference's impulse-response read-off including scipy.ndimage's drop of
 * taps with |w| <= DBL_EPSILON.  Host arithmetic (9 doubles per level). */
int kc_galerkin_coarsen(const double* w_fine9, int coarsening, double* w_coarse9);

/* Build the device hierarchy: GridState.__init__ (cycle.py:147-156) +
 * build_hierarchy (mesh.py:56-73).  w = n*9 doubles, stencil of level l at
 * w[9*(l-1) .. 9*(l-1)+8], w[dy+1][dx+1] row-major (stencil.py:66-70).
 * All v and f start at zero. */
int kc_create(int n, int coarsening, const double* w, int smoother_kind, double omega,
              int nu1, int nu2, int device, kc_handle** out);
int kc_destroy(kc_handle* h);
int kc_sync(kc_handle* h);

/* level data transfer: GridState.v[level-1] / f[level-1] item get/set */
int kc_level_dims(kc_handle* h, int level, int* nx, int* ny);
int kc_set(kc_handle* h, int level, int which, const double* host, long long ny, long long nx);
int kc_get(kc_handle* h, int level, int which, double* host, long long ny, long long nx);

/* state protocol (cycle.py:161-179), one call = one reference method */
int kc_relax(kc_handle* h, int level, int count);          /* relax_level, cycle.py:161-163 */
int kc_restrict_residual(kc_handle* h, int level);         /* restrict_residual, cycle.py:165-168 */
int kc_zero_guess(kc_handle* h, int level);                /* zero_guess, cycle.py:170-172 */
int kc_prolong_add(kc_handle* h, int level);               /* prolong_add, cycle.py:174-176 */
int kc_solve_coarsest(kc_handle* h);                       /* solve_coarsest, cycle.py:178-179 */

/* out = A v[level] (residual == 0; stencil.apply, stencil.py:108-113) or
 * out = f[level] - A v[level] (residual != 0; stencil.residual,
 * stencil.py:116-120) as a host (ny, nx) array.  Per-kernel parity entry
 * point; uses the level's free ping-pong buffer as scratch. */
int kc_apply(kc_handle* h, int level, int residual, double* out, long long ny, long long nx);

/* reductions (mesh.py:93-102), deterministic fixed-order fp64 */
int kc_norm2(kc_handle* h, int level, int which, double* out);
int kc_residual_norm(kc_handle* h, int level, double* out); /* ||f - A v|| (stencil.py:116-120) */

/* native kappa-cycle: run_cycle (cycle.py:261-263) executed `count` times as a
 * captured CUDA graph with fused kernels and the persistent bottom kernel. */
int kc_run_cycles(kc_handle* h, int kappa, int count);
/* same, bracketed by CUDA events on the handle's stream: bench_cycle
 * (cycle.py:381-410) timing of `count` back-to-back cycles in milliseconds. */
int kc_time_cycles(kc_handle* h, int kappa, int count, double* ms);

/* stand-alone solve loop (cycle.py:320-353) on the device.  v[1] must hold
 * the initial guess, f[1] the right-hand side.  err_hist/res_hist (may be
 * NULL) receive max_cycles+1 entries: index 0 is the initial norm.  Both
 * norms are recorded every cycle; stop_mode selects which one stops.
 * device_ms receives the CUDA-event time of the timed span (norm0 .. exit). */
int kc_solve(kc_handle* h, int kappa, int stop_mode, double target_reduction, int max_cycles,
             double* err_hist, double* res_hist, int* iterations, int* status, double* device_ms);

/* MGCG (krylov.py:60-141) on the device.  f and x0 are host arrays of the
 * finest interior shape (x0 may be NULL = zero start, krylov.py:74).  The
 * preconditioner is one kappa-cycle on (v = 0, f = r) (krylov.py:81-86); a
 * non-NULL `precond` replaces it (the reference's `precondition=` argument,
 * krylov.py:65): it receives r and must fill z, both host (ny, nx) arrays.
 * x_out (may be NULL) receives the final iterate.  hist (may be NULL)
 * receives up to max_it+1 values of the stop measure (||x|| for
 * KC_STOP_ERROR, recursive ||r|| for KC_STOP_RESIDUAL, krylov.py:88-89):
 * hist[0 .. iterations]; on a p.Ap breakdown (krylov.py:110-112) no measure
 * is taken at that step and hist[iterations] is NaN.
 * n_precond receives the number of preconditioner applications. */
typedef void (*kc_precond_fn)(const double* r, double* z, long long ny, long long nx, void* ctx);
int kc_pcg(kc_handle* h, int kappa, const double* f, const double* x0, int stop_mode,
           double target_reduction, int max_it, kc_precond_fn precond, void* ctx, double* hist,
           int* iterations, int* status, int* n_precond, double* x_out, double* device_ms);

/* Instrumentation: host-visible kernel launches and graph nodes of one
 * captured cycle (after kc_run_cycles/kc_solve built it). */
int kc_cycle_launches(kc_handle* h, int kappa, int* kernels_per_cycle);

/* Instrumentation: run ONE cycle eagerly (no graph) with a CUDA-event pair
 * around every scheduled op on the handle's stream; op_kind/op_level/op_arg/
 * op_ms receive up to max_ops entries (kinds: 0 relax, 1 restrict_residual,
 * 2 zero_guess, 3 prolong_add, 4 coarsest, 5 bottom sub-cycle).  Used for the
 * per-level cost fit of the run-time model and the
 * roofline of the fine-level kernels. */
int kc_profile_cycle(kc_handle* h, int kappa, int max_ops, int* op_kind, int* op_level, int* op_arg,
                     double* op_ms, int* n_ops);

/* the handle's CUDA stream (cudaStream_t as an opaque pointer) so a host
 * harness can record its own events on the stream the kernels run on */
int kc_stream(kc_handle* h, void** stream);

/* engine options: "fuse" (1: fused kernels in native cycles, the default;
 * 0: the per-op kernels) and "tile" (1: overlapped-tile kernels on sides
 * <= 511, the default; 0: streaming kernels there too), for A/B parity tests
 * and profiling.
 * Changing an option drops the captured graphs. */
int kc_set_option(kc_handle* h, const char* name, int value);

/* keep a device-resident copy of the finest v (kc_snapshot) and copy it back
 * (kc_restore): re-running a solve from the same start without host traffic */
int kc_snapshot(kc_handle* h);
int kc_restore(kc_handle* h);

/* v[level] (which = KC_WHICH_V) or f[level] = 0 on the device */
int kc_fill_zero(kc_handle* h, int level, int which);

/* ---------------------------------------------------------------------
 * Row-strip kernels for the multi-GPU decomposition.
 * Device pointers address the strip's interior origin (local row 0,
 * column 0); rows -2..-1 and ny..ny+1 are halo / zero ghost rows owned by
 * the caller; `stream` is a cudaStream_t (NULL = legacy stream).  Each call
 * is one reference operation on the strip, bit-identical to the
 * single-domain kernels.  w9 is the level stencil (host array of 9).
 * --------------------------------------------------------------------- */
int kc_strip_jacobi(const double* u, const double* f, double* out, int ny, int nx, int pitch, const double* w9,
                    double omega, int zero_u, void* stream);                        /* smoother.py:95-100 */
int kc_strip_resid_restrict(const double* u, const double* f, double* fc, int ncy, int ncx, int pitch,
                            int pitch_c, const double* w9, int zero_u, void* stream);  /* cycle.py:165-168 */
int kc_strip_prolong_add(double* v, const double* vc, int ny, int nx, int pitch, int pitch_c, int v_zero,
                         void* stream);                                                /* cycle.py:174-176 */
/* out (device, 2 doubles) = { sum v^2, sum (f - A v)^2 } over the strip's own rows */
int kc_strip_norms(const double* v, const double* f, int ny, int nx, int pitch, const double* w9, double* out,
                   void* stream);

/* Fused strip passes (the single-GPU k_pre / k_post on a strip): rows local
 * fine rows from global row gy0 (even) of mg, hb halo rows valid in the
 * buffers (>= nu1+2 for pre, >= nu2 for post; the caller exchanges them).
 * pre: nu1 sweeps of u (out in uo; nu1 = 0: uo untouched) + residual + full
 * weighting into fc for crows local coarse rows (cycle.py:211-213);
 * post: uo = relax^nu2(u + P vc) with vc's local row 0 at global coarse row
 * gy0/2, crows coarse rows and hbc (>= nu2/2 + 1) halo rows (cycle.py:219-220). */
int kc_strip_pre(const double* u, const double* f, double* uo, double* fc, int rows, int nx, int pitch, int pitch_c,
                 int crows, int gy0, int mg, int hb, const double* w9, double omega, int nu1, int zero_u,
                 void* stream);
int kc_strip_post(const double* u, const double* f, double* uo, const double* vc, int rows, int nx, int pitch,
                  int pitch_c, int crows, int gy0, int mg, int hb, int hbc, const double* w9, double omega, int nu2,
                  int v_zero, void* stream);
/* The same passes restricted to the coarse-row window [q_lo, q_hi) of the
 * chunk positions 0..crows (position crows carries a last rank's trailing
 * fine row): pre writes fc rows [q_lo, min(q_hi, crows)) and uo rows
 * [2 q_lo, min(2 q_hi, rows)); post writes uo rows [2 q_lo, min(2 q_hi, rows)).
 * hb / hbc may be as small as the rows the window's outputs depend on
 * (KC_EINVAL otherwise): a window of interior rows with hb = hbc = 0 never
 * touches the halo rows, so it runs while the caller's halo exchange is in
 * flight, and the boundary windows run after it (distributed.py overlap). */
int kc_strip_pre_window(const double* u, const double* f, double* uo, double* fc, int rows, int nx, int pitch,
                        int pitch_c, int crows, int gy0, int mg, int hb, int q_lo, int q_hi, const double* w9,
                        double omega, int nu1, int zero_u, void* stream);
int kc_strip_post_window(const double* u, const double* f, double* uo, const double* vc, int rows, int nx, int pitch,
                         int pitch_c, int crows, int gy0, int mg, int hb, int hbc, int q_lo, int q_hi,
                         const double* w9, double omega, int nu2, int v_zero, void* stream);

/* level data from / to device memory with an explicit row pitch (doubles):
 * agglomeration of distributed levels onto the native engine */
int kc_set_device(kc_handle* h, int level, int which, const double* dev, long long ny, long long nx,
                  long long pitch);
int kc_get_device(kc_handle* h, int level, int which, double* dev, long long ny, long long nx, long long pitch);
/* the same without waiting for the copy (ordered on the handle's stream) */
int kc_set_device_async(kc_handle* h, int level, int which, const double* dev, long long ny, long long nx,
                        long long pitch);
int kc_get_device_async(kc_handle* h, int level, int which, double* dev, long long ny, long long nx,
                        long long pitch);

/* issue all further work of the handle on `stream` (a cudaStream_t, NULL =
 * CUDA's stream 0; (void*)-1 = the handle's own stream again), e.g. a
 * framework's current stream, so the engine orders with the caller's kernels
 * and collectives */
int kc_set_stream(kc_handle* h, void* stream);

/* one kappa-cycle (kappa_cycle from level 1, cycle.py:204-220) issued op by op
 * on the handle's stream without waiting: capturable into the caller's CUDA
 * graph once the same cycle has run outside a capture */
int kc_cycle_enqueue(kc_handle* h, int kappa);

/* ---- device-side loops of the distributed solvers (distributed.py) ------
 * Every scalar of the reference's PCG loop (krylov.py:91-128) and
 * stand-alone loop (cycle.py:331-353) lives in a device array `scal` of
 * KC_DS_SLOTS doubles.  Strip kernels write per-rank partial sums into a
 * slot, the caller allreduces the slot in place (NCCL), and kc_dist_step
 * applies the reference's decisions on the device, so an iteration needs no
 * host read and a batch of iterations is one CUDA graph.  `part` is caller
 * scratch of KC_DS_PART doubles.  Once scal[KC_DS_DONE] is set the vector
 * updates are skipped. */
#define KC_DS_RZ 0
#define KC_DS_RZN 1
#define KC_DS_PAP 2
#define KC_DS_MEAS 3
#define KC_DS_ALPHA 4
#define KC_DS_BETA 5
#define KC_DS_TARGET 6
#define KC_DS_IT 7
#define KC_DS_MAXIT 8
#define KC_DS_STATUS 9        /* KC_STATUS_* once DONE */
#define KC_DS_DONE 10
#define KC_DS_JUST_DONE 11    /* set by the step that stopped the loop */
#define KC_DS_E2 12           /* stand-alone: sum v^2 (allreduced) */
#define KC_DS_R2 13           /* stand-alone: sum (f - A v)^2 (allreduced) */
#define KC_DS_STOP_RESIDUAL 14
#define KC_DS_STREAK 15
#define KC_DS_PREV 16
#define KC_DS_REDUCTION 17
#define KC_DS_SLOTS 32
#define KC_DS_PART 592
/* step kinds */
#define KC_DS_PCG_RZ0 0   /* rz = r.z of z = M r before the loop (krylov.py:100-104) */
#define KC_DS_PCG_PAP 1   /* it += 1; pAp breakdown or alpha = rz/pAp (krylov.py:107-113) */
#define KC_DS_PCG_MEAS 2  /* hist[it] = sqrt(meas); converged (krylov.py:116-120) */
#define KC_DS_PCG_RZ 3    /* rz_next breakdown, max_iterations, or beta = rz_next/rz, rz = rz_next (krylov.py:121-126) */
#define KC_DS_SOLVE 4     /* stand-alone norms of cycle it: stop / divergence rules (cycle.py:343-353) */

/* Ap = A p on the strip (p: one halo row each side) and the partial p.Ap
 * into scal[slot] (krylov.py:107-108, mesh.py:98-102) */
int kc_strip_apply_dot(const double* p, double* ap, int ny, int nx, int pitch, const double* w9, double* part,
                       double* scal, int slot, void* stream);
/* partial a.b into scal[slot] (mesh.py:98-102) */
int kc_strip_dot(const double* a, const double* b, int ny, int nx, int pitch, double* part, double* scal, int slot,
                 void* stream);
/* x += alpha p; r -= alpha ap (krylov.py:114-115) with alpha = scal[KC_DS_ALPHA];
 * partial of x.x (measure_x) or r.r into scal[KC_DS_MEAS] (krylov.py:88-89) */
int kc_strip_pcg_update_xr(double* x, double* r, const double* p, const double* ap, int ny, int nx, int pitch,
                           int measure_x, double* part, double* scal, void* stream);
/* p = z + beta p (krylov.py:125) with beta = scal[KC_DS_BETA] */
int kc_strip_pcg_update_p(double* p, const double* z, int ny, int nx, int pitch, const double* scal, void* stream);
/* r = f - A x (krylov.py:76); x carries one halo row each side */
int kc_strip_residual(const double* x, const double* f, double* r, int ny, int nx, int pitch, const double* w9,
                      void* stream);
/* dst = src when scal[KC_DS_JUST_DONE] (the stand-alone solution at the stop) */
int kc_strip_copy_if(const double* src, double* dst, int ny, int nx, int pitch, const double* scal, void* stream);
/* one scalar step of the loops (KC_DS_PCG_* / KC_DS_SOLVE); hist: PCG
 * measures hist[it], or stand-alone (error, residual) pairs hist[2it..2it+1] */
int kc_dist_step(int kind, double* scal, double* hist, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KCB200_H */
