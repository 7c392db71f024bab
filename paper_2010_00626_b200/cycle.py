"""kappa-cycles on the B200 engine (mirror of kcycle.cycle, cycle.py:1-410).

Two ways to run a cycle, both bit-identical to the reference's GridState:

* **drop-in (per-op)**: `CudaGridState` implements the reference's state
  protocol (cycle.py:114-179: `relax_level`, `restrict_residual`,
  `zero_guess`, `prolong_add`, `solve_coarsest`, `unknowns`, `n`, `nu1`,
  `nu2`, item access on `v`/`f`), each method one C-ABI call.  The
  reference's own `kcycle.cycle.kappa_cycle` / `run_cycle` can drive it
  unchanged, and so can `kappa_cycle` / `gamma_cycle` / `f_cycle` below.
* **native**: `run_cycle`, `solve_standalone`, `bench_cycle` and
  `krylov.pcg_solve` hand the whole cycle to the engine, which flattens the
  kappa recursion into fused HBM kernels plus a persistent shared-memory
  bottom kernel and replays it as one CUDA graph per cycle.  `CycleStats`
  are synthesized exactly from a dry run of the same recursion (the
  schedule is data independent), so they equal the reference's.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .mesh import Coarsening, HierarchySpec, build_hierarchy
from .smoother import SmootherKind, SmootherSpec
from .stencil import ProblemSpec, Stencil9, operator_hierarchy

__all__ = [
    "CycleConfig",
    "CycleStats",
    "SolveReport",
    "DryState",
    "CudaGridState",
    "GridState",
    "build_state",
    "kappa_cycle",
    "gamma_cycle",
    "f_cycle",
    "run_cycle",
    "solve_standalone",
    "bench_cycle",
    "BenchResult",
    "CONVERGED",
    "DIVERGED",
    "MAX_CYCLES",
    "BREAKDOWN",
]

CONVERGED = "converged"
DIVERGED = "diverged"
MAX_CYCLES = "max_cycles"
BREAKDOWN = "breakdown"


@dataclass(frozen=True)
class CycleConfig:
    """Cycle shape and smoothing configuration (cycle.py:53-82)."""

    n: int
    kappa: int | float = 1
    nu1: int = 2
    nu2: int = 2
    smoother: SmootherSpec = SmootherSpec(SmootherKind.DAMPED_JACOBI, omega=0.8)
    coarsening: Coarsening = Coarsening.FULL_STANDARD
    gamma: int = 1
    coarse_op: str = "galerkin"

    def __post_init__(self):
        if self.n < 1:
            raise ValueError(f"level count must be >= 1, got {self.n}")
        if self.kappa != math.inf and (self.kappa < 1 or int(self.kappa) != self.kappa):
            raise ValueError(f"kappa must be a positive integer or inf, got {self.kappa}")
        if self.gamma < 1:
            raise ValueError(f"gamma must be >= 1, got {self.gamma}")
        if self.nu1 < 0 or self.nu2 < 0:
            raise ValueError("relaxation counts must be >= 0")

    @property
    def effective_kappa(self) -> int:
        return self.n if self.kappa == math.inf else int(self.kappa)


@dataclass
class CycleStats:
    """Execution instrumentation accumulated across routine calls (cycle.py:85-111)."""

    visits: list[int]
    kernel_launches: int = 0
    unknown_touches: float = 0.0
    trace: list[tuple[int, int]] = field(default_factory=list)

    @classmethod
    def for_levels(cls, n: int) -> "CycleStats":
        return cls(visits=[0] * n)

    def record_call(self, level: int, counter: int, unknowns: int, coarsest: bool, nu: int):
        self.visits[level - 1] += 1
        self.trace.append((level, counter))
        if coarsest:
            self.kernel_launches += 1
        else:
            self.kernel_launches += 5 + nu
        self.unknown_touches += unknowns

    def absorb(self, other: "CycleStats", times: int = 1):
        """Add `times` repetitions of `other` (as if its calls were recorded again)."""
        if times <= 0:
            return
        for i, c in enumerate(other.visits):
            self.visits[i] += c * times
        self.kernel_launches += other.kernel_launches * times
        for _ in range(times):  # same float accumulation order as record_call
            self.unknown_touches += other.unknown_touches
        self.trace.extend(other.trace * times)

    def level_sequence(self) -> list[int]:
        return [level for level, _ in self.trace]

    def counter_sequence(self) -> list[int]:
        return [counter for _, counter in self.trace]


class DryState:
    """Recursion-only stand-in (cycle.py:114-141)."""

    def __init__(self, n: int, nu1: int = 0, nu2: int = 0,
                 coarsening: Coarsening = Coarsening.FULL_STANDARD):
        self.spec = build_hierarchy(n, coarsening)
        self.n = n
        self.nu1 = nu1
        self.nu2 = nu2

    def unknowns(self, level: int) -> int:
        return self.spec.unknowns(level)

    def relax_level(self, level: int, count: int):
        pass

    def restrict_residual(self, level: int):
        pass

    def zero_guess(self, level: int):
        pass

    def prolong_add(self, level: int):
        pass

    def solve_coarsest(self):
        pass


class _LevelData:
    """`state.v[i]` / `state.f[i]`: host copies in, host copies out (cycle.py:155-156)."""

    def __init__(self, state: "CudaGridState", which: int):
        self._s = state
        self._which = which

    def __len__(self):
        return self._s.n

    def _level(self, i: int) -> int:
        n = self._s.n
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError(f"level index {i} out of range")
        return i + 1

    def __getitem__(self, i: int) -> np.ndarray:
        level = self._level(i)
        nx, ny = self._s.spec.dims[level - 1]
        out = np.empty((ny, nx))
        self._s._check(self._s._lib.kc_get(self._s._h, level, self._which, N.dptr(out), ny, nx))
        return out

    def __setitem__(self, i: int, value) -> None:
        level = self._level(i)
        nx, ny = self._s.spec.dims[level - 1]
        a = N.as_f64c(value)
        if a.shape != (ny, nx):
            raise ValueError(f"dimension mismatch: {a.shape} vs {(ny, nx)}")
        self._s._check(self._s._lib.kc_set(self._s._h, level, self._which, N.dptr(a), ny, nx))


class CudaGridState:
    """Per-level (v, f, A) data of one solve, resident in HBM (GridState, cycle.py:144-179).

    The engine handle owns all device memory; the caller owns host arrays and
    copies happen at the boundary only (SURVEY.md §8(b) "Ownership").
    """

    def __init__(self, spec: HierarchySpec, ops: list[Stencil9], smoother: SmootherSpec,
                 nu1: int, nu2: int, device: int = 0, arith: str | None = None):
        if len(ops) != spec.n:
            raise ValueError(f"need {spec.n} operators, got {len(ops)}")
        self.spec = spec
        self.n = spec.n
        self.ops = ops
        self.smoother = smoother
        self.nu1 = nu1
        self.nu2 = nu2
        self.device = device
        self._h = None
        # "exact": libkcb200.so, iterates bit-identical to the reference;
        # "fast": libkcb200_fast.so, FMA-contracted (histories within 1e-10,
        # identical iteration counts); default N.default_arith()
        self.arith = N.default_arith() if arith is None else arith
        self._lib = N.lib_for(self.arith)
        w = np.ascontiguousarray(np.concatenate([op.w.ravel() for op in ops]), dtype=np.float64)
        h = C.c_void_p()
        N.check(self._lib.kc_create(spec.n, N.COARSENING_KIND[spec.coarsening.value], N.dptr(w),
                                N.SMOOTHER_KIND[smoother.kind.value], float(smoother.omega), nu1, nu2, device,
                                C.byref(h)), None, self._lib)
        self._h = h
        self.v = _LevelData(self, N.KC_WHICH_V)
        self.f = _LevelData(self, N.KC_WHICH_F)
        self._stats_cache: dict[int, CycleStats] = {}

    # -- lifetime ---------------------------------------------------------
    def close(self):
        if self._h is not None:
            self._lib.kc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int) -> None:
        N.check(rc, self._h, self._lib)

    # -- state protocol (cycle.py:158-179) ---------------------------------
    def unknowns(self, level: int) -> int:
        return self.spec.unknowns(level)

    def relax_level(self, level: int, count: int):
        self._check(self._lib.kc_relax(self._h, level, count))

    def restrict_residual(self, level: int):
        self._check(self._lib.kc_restrict_residual(self._h, level))

    def zero_guess(self, level: int):
        self._check(self._lib.kc_zero_guess(self._h, level))

    def prolong_add(self, level: int):
        self._check(self._lib.kc_prolong_add(self._h, level))

    def solve_coarsest(self):
        self._check(self._lib.kc_solve_coarsest(self._h))

    # -- device reductions / parity entry points ---------------------------
    def norm2(self, level: int = 1, which: str = "v") -> float:
        out = C.c_double()
        w = N.KC_WHICH_V if which == "v" else N.KC_WHICH_F
        self._check(self._lib.kc_norm2(self._h, level, w, C.byref(out)))
        return out.value

    def residual_norm(self, level: int = 1) -> float:
        out = C.c_double()
        self._check(self._lib.kc_residual_norm(self._h, level, C.byref(out)))
        return out.value

    def apply_level(self, level: int = 1, residual: bool = False) -> np.ndarray:
        nx, ny = self.spec.dims[level - 1]
        out = np.empty((ny, nx))
        self._check(self._lib.kc_apply(self._h, level, 1 if residual else 0, N.dptr(out), ny, nx))
        return out

    # -- native cycle --------------------------------------------------------
    def cycle_stats(self, kappa: int) -> CycleStats:
        """Exact per-cycle CycleStats of kappa_cycle(1, kappa) (data independent)."""
        st = self._stats_cache.get(kappa)
        if st is None:
            st = CycleStats.for_levels(self.n)
            kappa_cycle(DryState(self.n, self.nu1, self.nu2, self.spec.coarsening), 1, kappa, st)
            self._stats_cache[kappa] = st
        return st

    def run_cycles(self, kappa: int, count: int = 1):
        self._check(self._lib.kc_run_cycles(self._h, int(kappa), int(count)))

    def time_cycles(self, kappa: int, count: int = 1) -> float:
        ms = C.c_double()
        self._check(self._lib.kc_time_cycles(self._h, int(kappa), int(count), C.byref(ms)))
        return ms.value

    def launches_per_cycle(self, kappa: int) -> int:
        k = C.c_int()
        self._check(self._lib.kc_cycle_launches(self._h, int(kappa), C.byref(k)))
        return k.value

    def sync(self):
        self._check(self._lib.kc_sync(self._h))

    def stream_ptr(self) -> int:
        """cudaStream_t of the handle (for torch.cuda.ExternalStream timing)."""
        p = C.c_void_p()
        self._check(self._lib.kc_stream(self._h, C.byref(p)))
        return p.value or 0

    def solve_device(self, kappa: int, stop: str = "error", target_reduction: float = 1e8,
                     max_cycles: int = 10000):
        """kc_solve on the current v[0]/f[0]: (iterations, status, device_ms, err_hist, res_hist)."""
        err = np.zeros(max_cycles + 1)
        res = np.zeros(max_cycles + 1)
        it, st, dms = C.c_int(), C.c_int(), C.c_double()
        self._check(self._lib.kc_solve(self._h, int(kappa), N.KC_STOP_ERROR if stop == "error" else N.KC_STOP_RESIDUAL,
                                       float(target_reduction), int(max_cycles), N.dptr(err), N.dptr(res),
                                       C.byref(it), C.byref(st), C.byref(dms)))
        k = it.value
        return k, N.STATUS_NAMES[st.value], dms.value, err[: k + 1].tolist(), res[: k + 1].tolist()

    def get_level(self, level: int = 1, which: str = "v", out: np.ndarray | None = None) -> np.ndarray:
        """Copy v or f of `level` to the host (into `out` when given)."""
        nx, ny = self.spec.dims[level - 1]
        if out is None:
            out = np.empty((ny, nx))
        elif out.shape != (ny, nx) or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float64 array of the level shape")
        w = N.KC_WHICH_V if which == "v" else N.KC_WHICH_F
        self._check(self._lib.kc_get(self._h, level, w, N.dptr(out), ny, nx))
        return out

    def set_option(self, name: str, value: int):
        """Engine option (kc_set_option): "fuse" = 0 runs native cycles on the per-op kernels."""
        self._check(self._lib.kc_set_option(self._h, name.encode(), int(value)))

    def snapshot(self):
        """Keep a device copy of the finest v (restore() puts it back)."""
        self._check(self._lib.kc_snapshot(self._h))

    def restore(self):
        self._check(self._lib.kc_restore(self._h))

    def fill_zero(self, level: int = 1, which: str = "f"):
        self._check(self._lib.kc_fill_zero(self._h, level, N.KC_WHICH_F if which == "f" else N.KC_WHICH_V))

    OP_NAMES = ("relax", "restrict_residual", "zero_guess", "prolong_add", "coarsest", "bottom", "pre", "post",
                "postpre")

    def profile_cycle(self, kappa: int) -> list[dict]:
        """One eager cycle with CUDA events around every scheduled op."""
        cap = 1 << 16
        kind = (C.c_int * cap)()
        lev = (C.c_int * cap)()
        arg = (C.c_int * cap)()
        ms = (C.c_double * cap)()
        nops = C.c_int()
        self._check(self._lib.kc_profile_cycle(self._h, int(kappa), cap, kind, lev, arg, ms, C.byref(nops)))
        return [{"op": self.OP_NAMES[kind[i]], "level": lev[i], "arg": arg[i], "ms": ms[i]}
                for i in range(min(nops.value, cap))]


GridState = CudaGridState


def build_state(problem: ProblemSpec, config: CycleConfig, device: int = 0,
                arith: str | None = None) -> CudaGridState:
    """Hierarchy dims and per-level operators for one solve (cycle.py:266-270).
    `arith`: "exact" (bit-identical) or "fast" (FMA); default N.default_arith()."""
    spec = build_hierarchy(config.n, config.coarsening)
    ops = operator_hierarchy(problem, spec, config.coarse_op)
    return CudaGridState(spec, ops, config.smoother, config.nu1, config.nu2, device=device, arith=arith)


# ---------------------------------------------------------------------------
# recursions (per-op drivers of any state object)
# ---------------------------------------------------------------------------

def kappa_cycle(state, level: int, kappa: int, stats: CycleStats):
    """One counter-driven cycle starting at `level` (Algorithm 3; cycle.py:204-220)."""
    if kappa < 1:
        raise ValueError(f"cycle counter must be >= 1, got {kappa}")
    coarsest = level == state.n
    stats.record_call(level, kappa, state.unknowns(level), coarsest, state.nu1 + state.nu2)
    if coarsest:
        state.solve_coarsest()
        return
    state.relax_level(level, state.nu1)
    state.restrict_residual(level)
    state.zero_guess(level + 1)
    kappa_cycle(state, level + 1, kappa, stats)
    if kappa > 1:
        kappa_cycle(state, level + 1, kappa - 1, stats)
    state.prolong_add(level)
    state.relax_level(level, state.nu2)


def gamma_cycle(state, level: int, gamma: int, stats: CycleStats):
    """Classical cycle-index form (Algorithm 1; cycle.py:223-238)."""
    if gamma < 1:
        raise ValueError(f"gamma must be >= 1, got {gamma}")
    coarsest = level == state.n
    stats.record_call(level, gamma, state.unknowns(level), coarsest, state.nu1 + state.nu2)
    if coarsest:
        state.solve_coarsest()
        return
    state.relax_level(level, state.nu1)
    state.restrict_residual(level)
    state.zero_guess(level + 1)
    for _ in range(gamma):
        gamma_cycle(state, level + 1, gamma, stats)
    state.prolong_add(level)
    state.relax_level(level, state.nu2)


def f_cycle(state, level: int, stats: CycleStats):
    """Classical F form (Algorithm 2; cycle.py:241-258)."""
    coarsest = level == state.n
    stats.record_call(level, 2, state.unknowns(level), coarsest, state.nu1 + state.nu2)
    if coarsest:
        state.solve_coarsest()
        return
    state.relax_level(level, state.nu1)
    state.restrict_residual(level)
    state.zero_guess(level + 1)
    f_cycle(state, level + 1, stats)
    gamma_cycle(state, level + 1, 1, stats)
    state.prolong_add(level)
    state.relax_level(level, state.nu2)


def run_cycle(state, config: CycleConfig, stats: CycleStats):
    """One top-level cycle (cycle.py:261-263).  Native graph on a CudaGridState."""
    kappa = config.effective_kappa
    if isinstance(state, CudaGridState):
        state.run_cycles(kappa, 1)
        stats.absorb(state.cycle_stats(kappa))
    else:
        kappa_cycle(state, 1, kappa, stats)


# ---------------------------------------------------------------------------
# outer drivers
# ---------------------------------------------------------------------------

@dataclass
class SolveReport:
    """Outcome of an outer solve loop (cycle.py:281-293), plus device extras."""

    status: str
    iterations: int
    initial_error_norm: float
    final_error_norm: float
    per_cycle_reduction: list[float]
    asymptotic_factor: float | None
    stats: CycleStats
    wall_time_ms: float
    solution: np.ndarray | None = None
    # extras (not in the reference): full histories and the device-timed span
    error_history: list[float] | None = None
    residual_history: list[float] | None = None
    stop: str = "error"
    device_time_ms: float | None = None


def _asymptotic_factor(reductions: list[float], window: int = 5) -> float | None:
    tail = reductions[-window:]
    if not tail or any(r <= 0.0 for r in tail):
        return None
    return float(math.exp(sum(math.log(r) for r in tail) / len(tail)))


def _reductions(hist: list[float]) -> list[float]:
    return [hist[i] / hist[i - 1] if hist[i - 1] > 0.0 else 0.0 for i in range(1, len(hist))]


def _check_state_matches(state: CudaGridState, problem: ProblemSpec, config: CycleConfig) -> None:
    """A caller-supplied state must be the hierarchy build_state(problem,
    config) would make; a mismatch would silently solve another system."""
    if not isinstance(state, CudaGridState):
        raise TypeError("state must be a CudaGridState")
    if state.n != config.n or state.spec.coarsening != config.coarsening:
        raise ValueError(f"state hierarchy (n={state.n}, {state.spec.coarsening}) does not match the config "
                         f"(n={config.n}, {config.coarsening})")
    if (state.nu1, state.nu2) != (config.nu1, config.nu2):
        raise ValueError(f"state relaxation counts {(state.nu1, state.nu2)} != config {(config.nu1, config.nu2)}")
    if state.smoother != config.smoother:
        raise ValueError(f"state smoother {state.smoother} != config {config.smoother}")
    want = operator_hierarchy(problem, state.spec, config.coarse_op)
    if any(not np.array_equal(a.w, b.w) for a, b in zip(state.ops, want)):
        raise ValueError("state operators do not match the problem (epsilon, phi, coarse_op)")


def solve_standalone(
    problem: ProblemSpec,
    config: CycleConfig,
    target_reduction: float = 1e8,
    max_cycles: int = 10000,
    initial_guess: np.ndarray | None = None,
    *,
    stop: str = "error",
    device: int = 0,
    state: CudaGridState | None = None,
    solution_out: np.ndarray | None = None,
) -> SolveReport:
    """Repeated cycles on the zero-solution problem (cycle.py:303-366), on the device.

    `stop="error"` is the reference rule (||v_k|| <= ||v_0|| / target,
    cycle.py:332-347); `stop="residual"` stops on the true relative residual
    ||f - A v_k|| <= ||f - A v_0|| / target (BASELINE headline).  Both
    histories are recorded every cycle either way.  `state` lets a caller
    reuse an already built hierarchy (it must match `config`);
    `solution_out` (a C-contiguous float64 array of the finest shape, e.g.
    in pinned memory) receives the solution instead of a new array.
    """
    if target_reduction <= 1.0:
        raise ValueError(f"target reduction must exceed 1, got {target_reduction}")
    if stop not in ("error", "residual"):
        raise ValueError(f"stop must be 'error' or 'residual', got {stop!r}")
    fresh = state is None
    if fresh:
        state = build_state(problem, config, device=device)
    else:
        _check_state_matches(state, problem, config)
    nx, ny = state.spec.dims[0]
    if initial_guess is None:
        v0 = np.random.default_rng(problem.seed).random((ny, nx))
    else:
        if initial_guess.shape != (ny, nx):
            raise ValueError(f"initial guess shape {initial_guess.shape} != {(ny, nx)}")
        v0 = N.as_f64c(initial_guess)  # the upload is the reference's defensive copy
    state.v[0] = v0
    if not fresh:  # a fresh hierarchy starts with f = 0 on every level
        state.fill_zero(1, "f")
    kappa = config.effective_kappa
    state.launches_per_cycle(kappa)  # capture the cycle graph outside the timed span

    t0 = time.perf_counter()
    k, status, dev_ms, err_hist, res_hist = state.solve_device(kappa, stop, target_reduction, max_cycles)
    wall_ms = (time.perf_counter() - t0) * 1e3
    stats = CycleStats.for_levels(config.n)
    stats.absorb(state.cycle_stats(kappa), k)
    reductions = _reductions(err_hist if stop == "error" else res_hist)
    return SolveReport(
        status=status,
        iterations=k,
        initial_error_norm=err_hist[0],
        final_error_norm=err_hist[k],
        per_cycle_reduction=reductions,
        asymptotic_factor=_asymptotic_factor(reductions),
        stats=stats,
        wall_time_ms=wall_ms,
        solution=state.get_level(1, "v", solution_out),
        error_history=err_hist,
        residual_history=res_hist,
        stop=stop,
        device_time_ms=dev_ms,
    )


@dataclass(frozen=True)
class BenchResult:
    """Single-cycle benchmark cell (cycle.py:369-378)."""

    kappa: int | float
    n: int
    mean_ms: float | None
    launches: int
    op_units: float


def bench_cycle(problem: ProblemSpec, config: CycleConfig, reps: int, device: int = 0) -> BenchResult:
    """Time `reps` single cycles on fixed random data (cycle.py:381-410).

    Each repetition restores v[0] = v0 (untimed) and times one cycle with CUDA
    events on the handle's stream.  reps = 0 is a dry run (counts only).
    """
    if reps < 0:
        raise ValueError(f"reps must be >= 0, got {reps}")
    counts = CycleStats.for_levels(config.n)
    if reps == 0:
        dry = DryState(config.n, config.nu1, config.nu2, config.coarsening)
        kappa_cycle(dry, 1, config.effective_kappa, counts)
        return BenchResult(config.kappa, config.n, None, counts.kernel_launches, counts.unknown_touches)
    state = build_state(problem, config, device=device)
    v0 = np.random.default_rng(problem.seed).random(state.v[0].shape)
    kappa = config.effective_kappa
    state.v[0] = v0
    state.run_cycles(kappa, 1)  # warm-up (also captures the graph)
    counts.absorb(state.cycle_stats(kappa))
    times = []
    for _ in range(reps):
        state.v[0] = v0
        times.append(state.time_cycles(kappa, 1))
    state.close()
    return BenchResult(config.kappa, config.n, float(np.mean(times)), counts.kernel_launches,
                       counts.unknown_touches)
