"""Cycle-preconditioned CG on the device (mirror of kcycle.krylov, krylov.py:1-141).

Standard (non-flexible) PCG; M^-1 r = one kappa-cycle on (v = 0, f = r)
(krylov.py:81-86), executed as the engine's captured cycle graph.  The
residual r lives in the finest level's f buffer and z is the finest v, so a
preconditioner application moves no data.  Vector updates are fused kernels
with the reference's rounding (kc_pcg.cuh); only the dot products are
reordered (deterministic tree instead of OpenBLAS ddot).
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .cycle import CycleConfig, CycleStats, CudaGridState, SolveReport, _asymptotic_factor, _reductions

__all__ = ["PcgConfig", "pcg_solve"]


@dataclass(frozen=True)
class PcgConfig:
    """Preconditioned CG settings (krylov.py:39-57)."""

    cycle: CycleConfig
    target_reduction: float = 1e8
    max_iterations: int = 10000
    stop: str = "residual"

    def __post_init__(self):
        if self.target_reduction <= 1.0:
            raise ValueError(f"target reduction must exceed 1, got {self.target_reduction}")
        if self.stop not in ("error", "residual"):
            raise ValueError(f"stop must be 'error' or 'residual', got {self.stop!r}")


def pcg_solve(state: CudaGridState, f: np.ndarray, config: PcgConfig, x0: np.ndarray | None = None,
              precondition=None) -> SolveReport:
    """Preconditioned CG on the finest-level system of `state` (krylov.py:60-141).

    `precondition`, when given, replaces the cycle: a host callable r -> z
    (the reference's test hook, krylov.py:65, 81).
    """
    if not isinstance(state, CudaGridState):
        raise TypeError("pcg_solve needs a CudaGridState (device-resident hierarchy)")
    nx, ny = state.spec.dims[0]
    fa = N.as_f64c(f)
    if fa.shape != (ny, nx):
        raise ValueError(f"dimension mismatch: {fa.shape} vs {(ny, nx)}")
    xa = None if x0 is None else N.as_f64c(np.asarray(x0, dtype=float))
    if xa is not None and xa.shape != (ny, nx):
        raise ValueError(f"dimension mismatch: {xa.shape} vs {(ny, nx)}")
    kappa = config.cycle.effective_kappa
    mi = int(config.max_iterations)
    hist = np.zeros(mi + 1)
    xout = np.empty((ny, nx))
    it, st, napp, dms = C.c_int(), C.c_int(), C.c_int(), C.c_double()

    errors: list[BaseException] = []
    cb = N.PRECOND_FN()  # NULL
    if precondition is not None:
        def _cb(r_ptr, z_ptr, ny_, nx_, _ctx):
            try:
                r = np.ctypeslib.as_array(r_ptr, shape=(ny_, nx_)).copy()
                z = N.as_f64c(precondition(r))
                np.ctypeslib.as_array(z_ptr, shape=(ny_, nx_))[...] = z
            except BaseException as exc:  # surfaced after the call returns
                errors.append(exc)
                # NaN makes r . z fail the rz > 0 test at once (breakdown)
                np.ctypeslib.as_array(z_ptr, shape=(ny_, nx_))[...] = np.nan
        cb = N.PRECOND_FN(_cb)
    else:
        state.launches_per_cycle(kappa)  # capture outside the timed span

    t0 = time.perf_counter()
    rc = state._lib.kc_pcg(state._h, kappa, N.dptr(fa), None if xa is None else N.dptr(xa),
                      N.KC_STOP_ERROR if config.stop == "error" else N.KC_STOP_RESIDUAL,
                      float(config.target_reduction), mi, cb, None, N.dptr(hist),
                      C.byref(it), C.byref(st), C.byref(napp), N.dptr(xout), C.byref(dms))
    wall_ms = (time.perf_counter() - t0) * 1e3
    if errors:
        raise errors[0]
    N.check(rc, state._h, state._lib)
    k = it.value
    status = N.STATUS_NAMES[st.value]
    # a p.Ap breakdown at step k took no measure there (krylov.py:110-112):
    # the engine marks hist[k] NaN; an r.z breakdown came after measuring
    nh = k + 1
    if status == "breakdown" and k > 0 and math.isnan(hist[k]):
        nh = k
    h = hist[:nh].tolist()
    stats = CycleStats.for_levels(state.n)
    if precondition is None:
        stats.absorb(state.cycle_stats(kappa), napp.value)
    reductions = _reductions(h)
    return SolveReport(
        status=status,
        iterations=k,
        initial_error_norm=h[0],
        final_error_norm=h[-1],
        per_cycle_reduction=reductions,
        asymptotic_factor=_asymptotic_factor(reductions),
        stats=stats,
        wall_time_ms=wall_ms,
        solution=xout,
        error_history=h if config.stop == "error" else None,
        residual_history=h if config.stop == "residual" else None,
        stop=config.stop,
        device_time_ms=dms.value,
    )
