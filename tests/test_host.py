"""CPU-only tests: host logic of the package and the C-ABI library surface.

No CUDA compute here (there is no GPU in the build container): the library
must load, export every symbol include/kcb200.h declares, compute the
Galerkin setup bit-exactly (host C++), and refuse to run without a GPU.
"""

import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_json

kc = pytest.importorskip("paper_2010_00626_b200")
from paper_2010_00626_b200 import _native as N  # noqa: E402
from paper_2010_00626_b200 import (  # noqa: E402
    Coarsening, CycleConfig, CycleStats, DryState, PcgConfig, ProblemSpec, Stencil9, build_hierarchy,
    f_cycle, gamma_cycle, kappa_cycle, operator_hierarchy, rotated_anisotropic_stencil, run_cycle)
from paper_2010_00626_b200.smoother import SmootherKind, SmootherSpec  # noqa: E402

INF = math.inf


def header_symbols():
    src = open(os.path.join(ROOT, "include", "kcb200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(kc_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(N.lib, s), s
        assert s in N._SIGS, f"{s} declared in the header but not bound in _native"


def test_abi_version():
    assert N.lib.kc_abi_version() == 1


def test_fast_build_exports_the_same_abi():
    """libkcb200_fast.so (the FMA build of the same sources) loads, reports
    its arithmetic mode and exports every header symbol; the exact build
    reports exact."""
    fast = N.lib_for("fast")
    assert fast is not N.lib
    assert N.lib.kc_arith_mode() == 0 and fast.kc_arith_mode() == 1
    assert fast.kc_abi_version() == 1
    for s in header_symbols():
        assert hasattr(fast, s), s


def test_arith_selection(monkeypatch):
    assert N.lib_for("exact") is N.lib
    monkeypatch.setenv("KCB200_ARITH", "fast")
    assert N.default_arith() == "fast" and N.lib_for() is N.lib_for("fast")
    monkeypatch.setenv("KCB200_ARITH", "bogus")
    with pytest.raises(ValueError):
        N.default_arith()
    with pytest.raises(ValueError):
        N.lib_for("double")


def test_create_without_gpu_fails_loudly_in_both_builds():
    """No CPU fallback: without a device kc_create raises CudaUnavailableError
    (the package never routes through the oracle or numpy)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    for arith in ("exact", "fast"):
        with pytest.raises(kc.CudaUnavailableError):
            kc.build_state(ProblemSpec(1e-4, 45.0), CycleConfig(n=3), arith=arith)


def test_stencil_hand_values():
    """test_stencil.py:26-34: eps=0.1, phi=45 -> centre 2.2, edges -0.55, corners +-0.225."""
    w = rotated_anisotropic_stencil(0.1, 45.0).w
    assert w[1, 1] == pytest.approx(2.2)
    assert w[0, 1] == pytest.approx(-0.55) and w[1, 0] == pytest.approx(-0.55)
    assert w[0, 0] == pytest.approx(-0.225) and w[0, 2] == pytest.approx(0.225)


def test_galerkin_hierarchy_bit_exact_vs_reference(golden_stencils):
    for e in golden_stencils:
        ops = operator_hierarchy(ProblemSpec(e["epsilon"], e["phi"]),
                                 build_hierarchy(e["n"], Coarsening.FULL_STANDARD), e["coarse_op"])
        got = [[float(x).hex() for x in op.w.ravel()] for op in ops]
        assert got == e["w_hex"], (e["epsilon"], e["phi"], e["coarse_op"])


def test_galerkin_semi_y_symmetry():
    from paper_2010_00626_b200.stencil import galerkin_coarsen
    c = galerkin_coarsen(rotated_anisotropic_stencil(1.0, 0.0), Coarsening.SEMI_Y).w
    assert np.allclose(c, c[::-1, ::-1])
    assert abs(c.sum()) < 1e-14


def test_hierarchy_dims():
    assert build_hierarchy(3, Coarsening.FULL_STANDARD).dims == ((7, 7), (3, 3), (1, 1))
    assert build_hierarchy(3, Coarsening.SEMI_Y).dims == ((7, 7), (7, 3), (7, 1))
    with pytest.raises(ValueError):
        build_hierarchy(0, Coarsening.FULL_STANDARD)


def test_config_validation():
    with pytest.raises(ValueError):
        CycleConfig(n=0, kappa=1)
    with pytest.raises(ValueError):
        CycleConfig(n=3, kappa=0)
    with pytest.raises(ValueError):
        CycleConfig(n=3, kappa=2.5)
    with pytest.raises(ValueError):
        CycleConfig(n=3, kappa=1, nu1=-1)
    assert CycleConfig(n=3, kappa=INF).effective_kappa == 3
    with pytest.raises(ValueError):
        PcgConfig(cycle=CycleConfig(n=3), target_reduction=1.0)
    with pytest.raises(ValueError):
        PcgConfig(cycle=CycleConfig(n=3), stop="both")
    with pytest.raises(ValueError):
        SmootherSpec(SmootherKind.DAMPED_JACOBI, 1.5)
    with pytest.raises(ValueError):
        ProblemSpec(epsilon=0.0)


def test_dry_stats_match_reference():
    d = load_json("dry_stats.json")
    for key, rec in d.items():
        parts = key.split("_")
        n = int(parts[0][1:])
        kn = parts[1][1:]
        nu1, nu2 = int(parts[2][2]), int(parts[2][3])
        kappa = INF if kn == "W" else int(kn)
        st = CycleStats.for_levels(n)
        run_cycle(DryState(n, nu1, nu2), CycleConfig(n=n, kappa=kappa, nu1=nu1, nu2=nu2), st)
        assert st.visits == rec["visits"], key
        assert st.kernel_launches == rec["kernel_launches"], key
        assert st.unknown_touches == rec["unknown_touches"], key
        assert len(st.trace) == rec["trace_len"], key
        if "trace" in rec:
            assert [list(t) for t in st.trace] == rec["trace"], key


def test_absorb_equals_repeated_recording():
    n = 6
    one = CycleStats.for_levels(n)
    kappa_cycle(DryState(n, 2, 2), 1, 3, one)
    rep = CycleStats.for_levels(n)
    for _ in range(7):
        kappa_cycle(DryState(n, 2, 2), 1, 3, rep)
    agg = CycleStats.for_levels(n)
    agg.absorb(one, 7)
    assert agg == rep


def test_classical_forms_dry():
    s1, s2 = CycleStats.for_levels(4), CycleStats.for_levels(4)
    gamma_cycle(DryState(4), 1, 2, s1)
    assert s1.visits == [1, 2, 4, 8]
    f_cycle(DryState(4), 1, s2)
    assert s2.visits == [1, 2, 3, 4]


def test_no_gpu_fails_loudly():
    """The engine has no CPU fallback: without a device, building a state raises."""
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    from paper_2010_00626_b200 import build_state
    with pytest.raises(N.CudaUnavailableError):
        build_state(ProblemSpec(1e-4, 45.0), CycleConfig(n=3))


def test_zebra_and_semi_coarsening_reach_the_engine():
    """Zebra smoothers and y-semi-coarsening are engine paths now (§8(f)1): the
    Python layer passes them to kc_create, which without a GPU fails with
    CudaUnavailableError (never a silent CPU fallback) and on a B200 builds."""
    from paper_2010_00626_b200 import CudaUnavailableError
    from paper_2010_00626_b200.cycle import CudaGridState
    w = np.array([[0.1, -0.5, 0.1], [-0.5, 2.0, -0.5], [0.1, -0.5, 0.1]])
    for co, kind in ((Coarsening.SEMI_Y, SmootherKind.DAMPED_JACOBI), (Coarsening.FULL_STANDARD, SmootherKind.ZEBRA_X),
                     (Coarsening.SEMI_Y, SmootherKind.ZEBRA_ALTERNATING)):
        spec = build_hierarchy(3, co)
        try:
            CudaGridState(spec, [Stencil9(w)] * 3, SmootherSpec(kind), 2, 2).close()
        except CudaUnavailableError:
            pass
