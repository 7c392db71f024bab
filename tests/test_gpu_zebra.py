"""Zebra line relaxation and y-semi-coarsening on the B200 engine
(the paper's solvers 3-6) against the reference's own
outputs (tests/golden/zebra.npz, tests/golden/make_golden.py zebra).

The line solves restate LAPACK dgtsv (scipy.linalg.solve_banded) with the
elimination plan precomputed on the host and the same operand order, so the
bar is bit-identical iterates, as for the Jacobi path.
"""

import numpy as np
import pytest

from conftest import load_json, load_npz

from paper_2010_00626_b200 import (CycleConfig, CycleStats, ProblemSpec, build_state, run_cycle,
                                   solve_standalone)
from paper_2010_00626_b200.cycle import CudaGridState
from paper_2010_00626_b200.mesh import Coarsening, build_hierarchy
from paper_2010_00626_b200.smoother import SmootherKind, SmootherSpec
from paper_2010_00626_b200.stencil import Stencil9

pytestmark = pytest.mark.gpu

INF = float("inf")
Z = load_npz("zebra.npz")
META = load_json("zebra_meta.json")
SM = {"jacobi": SmootherKind.DAMPED_JACOBI, "zebra-x": SmootherKind.ZEBRA_X, "zebra-y": SmootherKind.ZEBRA_Y,
      "zebra-xy": SmootherKind.ZEBRA_ALTERNATING}
CO = {"full": Coarsening.FULL_STANDARD, "semi-y": Coarsening.SEMI_Y}


def _placement(ny, nx):
    """(coarsening, n, level) whose level has shape (ny, nx), or None."""
    if ny == nx:
        return Coarsening.FULL_STANDARD, int(nx + 1).bit_length() - 1, 1
    n = int(nx + 1).bit_length() - 1
    for level in range(1, n + 1):
        if 2 ** (n - level + 1) - 1 == ny:
            return Coarsening.SEMI_Y, n, level
    return None


def _state(co, n, w, kind):
    ops = [Stencil9(np.asarray(w))] * n
    return CudaGridState(build_hierarchy(n, co), ops, SmootherSpec(kind, 0.8), 0, 0)


@pytest.mark.parametrize("key", META["kernels"])
def test_zebra_kernels_bit_exact(key):
    u, f, w = Z[key + "_u"], Z[key + "_f"], Z[key + "_w"]
    place = _placement(*u.shape)
    if place is None:
        pytest.skip(f"shape {u.shape} is not a level of an engine hierarchy (oracle-tested)")
    co, n, level = place
    i = level - 1
    for kind, count, ref in ((SmootherKind.ZEBRA_X, 1, "_zx"), (SmootherKind.ZEBRA_Y, 1, "_zy"),
                             (SmootherKind.ZEBRA_ALTERNATING, 2, "_zxy2")):
        st = _state(co, n, w, kind)
        st.v[i], st.f[i] = u, f
        st.relax_level(level, count)
        assert np.array_equal(st.v[i], Z[key + ref]), (key, kind)
        st.close()
    if co is Coarsening.SEMI_Y and level < n:  # transfers into / out of the next semi-y level
        st = _state(co, n, w, SmootherKind.ZEBRA_X)
        st.f[i] = f
        st.zero_guess(level)
        st.restrict_residual(level)
        assert np.array_equal(st.f[i + 1], Z[key + "_rsemi"]), key
        st.close()
    if co is Coarsening.SEMI_Y and level > 1:
        st = _state(co, n, w, SmootherKind.ZEBRA_X)
        st.v[i] = u
        st.v[i - 1] = np.zeros(st.v[i - 1].shape)
        st.prolong_add(level - 1)
        assert np.array_equal(st.v[i - 1], Z[key + "_psemi"]), key
        st.close()
    if key + "_coarsest" in Z.files and co is Coarsening.SEMI_Y and level == n:
        st = _state(co, n, w, SmootherKind.ZEBRA_X)
        st.f[i] = f
        st.solve_coarsest()
        assert np.array_equal(st.v[i], Z[key + "_coarsest"]), key
        st.close()


@pytest.mark.parametrize("key", sorted(META["cycles"]))
def test_zebra_cycles_bit_exact(key):
    rec = META["cycles"][key]
    n = rec["n"]
    kappa = INF if rec["kappa"] == "W" else int(rec["kappa"])
    cfg = CycleConfig(n=n, kappa=kappa, smoother=SmootherSpec(SM[rec["smoother"]], 0.8),
                      coarsening=CO[rec["coarsening"]])
    st = build_state(ProblemSpec(0.5, 30.0), cfg)
    st.v[0], st.f[0] = Z[key + "_v0"], Z[key + "_f0"]
    stats = CycleStats.for_levels(n)
    for c in (1, 2):
        run_cycle(st, cfg, stats)
        assert np.array_equal(st.v[0], Z[f"{key}_c{c}"]), (key, c)
    assert stats.visits == rec["visits"]
    assert stats.kernel_launches == rec["kernel_launches"]
    st.close()


@pytest.mark.parametrize("key", sorted(META["solves"]))
def test_zebra_solves_match_reference(key):
    rec = META["solves"][key]
    cfg = CycleConfig(n=rec["n"], kappa=int(rec["kappa"]), smoother=SmootherSpec(SM[rec["smoother"]], 0.8),
                      coarsening=CO[rec["coarsening"]])
    rep = solve_standalone(ProblemSpec(1e-4, 45.0, seed=0), cfg, 1e8, max_cycles=2000)
    assert rep.status == rec["status"] and rep.iterations == rec["iterations"]
    assert rep.initial_error_norm == pytest.approx(rec["initial_error_norm"], rel=1e-12)
    assert rep.final_error_norm == pytest.approx(rec["final_error_norm"], rel=1e-10)
    assert rep.stats.kernel_launches == rec["kernel_launches"]
    assert rep.stats.unknown_touches == rec["unknown_touches"]


def test_pure_function_zebra_sweep_matches_reference():
    """kernels.zebra_line_sweep / relax (the reference's pure-function
    signatures) on square grids."""
    from paper_2010_00626_b200 import kernels as K
    for key in META["kernels"]:
        u = Z[key + "_u"]
        if u.shape[0] != u.shape[1]:
            continue
        f, op = Z[key + "_f"], Stencil9(Z[key + "_w"])
        assert np.array_equal(K.zebra_line_sweep(op, u, f, "x"), Z[key + "_zx"]), key
        assert np.array_equal(K.zebra_line_sweep(op, u, f, "y"), Z[key + "_zy"]), key
        assert np.array_equal(K.relax(op, u, f, SmootherSpec(SmootherKind.ZEBRA_ALTERNATING), 2), Z[key + "_zxy2"])
