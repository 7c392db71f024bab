"""Level-hierarchy bookkeeping (mirror of kcycle.mesh, mesh.py:1-102).

Only the hierarchy description lives on the host; level data lives in HBM,
owned by a `CudaGridState` (cycle.py).  Sizes follow the reference exactly:
level l (1 = finest) of an n-level full-coarsening hierarchy has interior side
2**(n-l+1) - 1 (mesh.py:56-68).  The device stores each level with a zero
ghost ring and a 128-byte aligned pitch.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

__all__ = ["Coarsening", "HierarchySpec", "build_hierarchy"]


class Coarsening(Enum):
    """How the hierarchy shrinks from one level to the next (mesh.py:35-39)."""

    FULL_STANDARD = "full"
    SEMI_Y = "semi-y"


@dataclass(frozen=True)
class HierarchySpec:
    """Level count plus per-level interior sizes (nx, ny), finest first (mesh.py:42-53)."""

    n: int
    coarsening: Coarsening
    dims: tuple[tuple[int, int], ...]

    def unknowns(self, level: int) -> int:
        nx, ny = self.dims[level - 1]
        return nx * ny


def build_hierarchy(n: int, coarsening: Coarsening) -> HierarchySpec:
    """Dims for an n-level hierarchy whose finest side is 2**n - 1 (mesh.py:56-73)."""
    if n < 1:
        raise ValueError(f"level count must be >= 1, got {n}")
    if coarsening is Coarsening.FULL_STANDARD:
        dims = tuple((2 ** (n - l + 1) - 1, 2 ** (n - l + 1) - 1) for l in range(1, n + 1))
    elif coarsening is Coarsening.SEMI_Y:
        nx = 2 ** n - 1
        dims = tuple((nx, 2 ** (n - l + 1) - 1) for l in range(1, n + 1))
    else:
        raise ValueError(f"unknown coarsening kind: {coarsening!r}")
    return HierarchySpec(n=n, coarsening=coarsening, dims=dims)
