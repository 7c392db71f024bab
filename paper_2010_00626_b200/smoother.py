"""Relaxation configuration (mirror of kcycle.smoother's SmootherKind/SmootherSpec,
smoother.py:36-53).  The sweeps themselves run on the device: damped Jacobi
in the fused streaming / tile / bottom kernels (kc_stream.cuh, kc_tile.cuh,
kc_bottom.cuh), zebra x / y / alternating line relaxation in kc_zebra.cuh."""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

__all__ = ["SmootherKind", "SmootherSpec"]


class SmootherKind(Enum):
    DAMPED_JACOBI = "jacobi"
    ZEBRA_X = "zebra-x"
    ZEBRA_Y = "zebra-y"
    ZEBRA_ALTERNATING = "zebra-xy"


@dataclass(frozen=True)
class SmootherSpec:
    """Relaxation kind plus the Jacobi damping factor (smoother.py:44-53)."""

    kind: SmootherKind
    omega: float = 0.8

    def __post_init__(self):
        if self.kind is SmootherKind.DAMPED_JACOBI and not 0.0 < self.omega <= 1.0:
            raise ValueError(f"jacobi damping must lie in (0, 1], got {self.omega}")
