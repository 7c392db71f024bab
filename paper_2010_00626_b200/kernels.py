"""Device-backed pure functions with the reference's signatures (parity entry points).

Each function uploads its host inputs to a transient engine handle, runs the
one CUDA kernel that implements the reference operation and returns a new
host array; inputs are never modified (smoother.py:11-12, mesh.py:9-10).
Sides must be 2**k - 1 (the engine's level shapes).  These exist for
per-kernel parity tests and drop-in convenience; the solvers never call them.

  apply / residual       stencil.py:108-120      k_apply
  damped_jacobi_sweep    smoother.py:95-100      k_jacobi
  relax                  smoother.py:138-163     k_jacobi x count
  restrict               transfer.py:70-83       k_resid_restrict (zero u)
  prolong                transfer.py:46-58       k_prolong_add (zero v)
  coarsest_solve         cycle.py:182-200        k_coarsest / k_coarsest_line (semi-y)
  zebra_line_sweep       smoother.py:107-135     k_zebra_rhs_* + k_zebra_solve_*
  norm2 / dot-free norm  mesh.py:93-95           k_red_partial + k_red_final
"""

from __future__ import annotations

import numpy as np

from .cycle import CudaGridState
from .mesh import Coarsening, build_hierarchy
from .smoother import SmootherKind, SmootherSpec
from .stencil import Stencil9

__all__ = ["apply", "residual", "damped_jacobi_sweep", "relax", "restrict", "prolong",
           "coarsest_solve", "zebra_line_sweep", "norm2"]

_ID = Stencil9([[0.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 0.0]])


def _levels_for(side: int) -> int:
    n = int(side + 1).bit_length() - 1
    if side < 1 or (1 << n) - 1 != side:
        raise ValueError(f"engine level sides are 2**k - 1, got {side}")
    return n


def _state(side: int, ops_top: list[Stencil9], omega: float = 0.8,
           kind: SmootherKind = SmootherKind.DAMPED_JACOBI) -> CudaGridState:
    n = _levels_for(side)
    ops = list(ops_top) + [_ID] * (n - len(ops_top))
    return CudaGridState(build_hierarchy(n, Coarsening.FULL_STANDARD), ops[:n],
                         SmootherSpec(kind, omega if 0 < omega <= 1 else 0.8), 0, 0)


def _square(a) -> np.ndarray:
    a = np.asarray(a, dtype=float)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError(f"engine grids are square, got shape {a.shape}")
    return a


def apply(op: Stencil9, u) -> np.ndarray:
    u = _square(u)
    s = _state(u.shape[0], [op])
    s.v[0] = u
    out = s.apply_level(1)
    s.close()
    return out


def residual(op: Stencil9, u, f) -> np.ndarray:
    u, f = _square(u), _square(f)
    if u.shape != f.shape:
        raise ValueError(f"dimension mismatch: {u.shape} vs {f.shape}")
    s = _state(u.shape[0], [op])
    s.v[0] = u
    s.f[0] = f
    out = s.apply_level(1, residual=True)
    s.close()
    return out


def relax(op: Stencil9, u, f, spec: SmootherSpec, count: int) -> np.ndarray:
    if count < 0:
        raise ValueError(f"relaxation count must be >= 0, got {count}")
    if spec.kind is SmootherKind.ZEBRA_ALTERNATING and count % 2:
        raise ValueError("alternating zebra needs an even relaxation count")
    if spec.kind is SmootherKind.DAMPED_JACOBI and op.center == 0.0 and count > 0:
        raise ValueError("zero center coefficient")
    u, f = _square(u), _square(f)
    if u.shape != f.shape:
        raise ValueError(f"dimension mismatch: {u.shape} vs {f.shape}")
    s = _state(u.shape[0], [op], spec.omega, spec.kind)
    s.v[0] = u
    s.f[0] = f
    s.relax_level(1, count)
    out = s.v[0]
    s.close()
    return out


def damped_jacobi_sweep(op: Stencil9, u, f, omega: float) -> np.ndarray:
    return relax(op, u, f, SmootherSpec(SmootherKind.DAMPED_JACOBI, omega), 1)


def restrict(fine, kind: Coarsening = Coarsening.FULL_STANDARD) -> np.ndarray:
    if kind is not Coarsening.FULL_STANDARD:
        raise ValueError("the B200 engine implements full coarsening only")
    fine = _square(fine)
    if fine.shape[0] < 3 or fine.shape[0] % 2 == 0:
        raise ValueError(f"fine ny must be odd and >= 3, got {fine.shape[0]}")
    s = _state(fine.shape[0], [_ID])
    s.f[0] = fine
    s.zero_guess(1)           # r = f - A*0 = f exactly
    s.restrict_residual(1)
    out = s.f[1]
    s.close()
    return out


def prolong(coarse, kind: Coarsening = Coarsening.FULL_STANDARD) -> np.ndarray:
    if kind is not Coarsening.FULL_STANDARD:
        raise ValueError("the B200 engine implements full coarsening only")
    coarse = _square(coarse)
    s = _state(2 * coarse.shape[0] + 1, [_ID])
    s.v[1] = coarse
    s.zero_guess(1)           # v = 0 + P vc
    s.prolong_add(1)
    out = s.v[0]
    s.close()
    return out


def coarsest_solve(op: Stencil9, f, coarsening: Coarsening = Coarsening.FULL_STANDARD) -> np.ndarray:
    f = np.asarray(f, dtype=float)
    if f.shape != (1, 1):
        raise ValueError(f"not a coarsest grid for {coarsening}: shape {f.shape}")
    s = _state(1, [op])
    s.f[0] = f
    s.solve_coarsest()
    out = s.v[0]
    s.close()
    return out


def zebra_line_sweep(op: Stencil9, u, f, axis: str) -> np.ndarray:
    """One zebra sweep with lines along `axis` (smoother.py:107-135)."""
    if axis not in ("x", "y"):
        raise ValueError(f"axis must be 'x' or 'y', got {axis!r}")
    kind = SmootherKind.ZEBRA_X if axis == "x" else SmootherKind.ZEBRA_Y
    return relax(op, u, f, SmootherSpec(kind), 1)


def norm2(g) -> float:
    g = _square(g)
    s = _state(g.shape[0], [_ID])
    s.v[0] = g
    out = s.norm2(1)
    s.close()
    return out
