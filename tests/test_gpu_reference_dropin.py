"""The drop-in proof with the REAL reference code.

The unmodified reference package `kcycle` (installed into the git-ignored
baseline/_ref by tools/install_reference.sh; it travels to the GPU box with
the snapshot) drives this repo's `CudaGridState` through its own cycle
drivers and solvers:

* `kcycle.cycle.kappa_cycle` / `gamma_cycle` / `f_cycle` / `run_cycle`
  (cycle.py:204-263) on a CudaGridState vs the same calls on the
  reference's own numpy `GridState`: iterates bit-identical, CycleStats
  identical, n = 5 / 7 / 9, every kappa;
* `kcycle.krylov.pcg_solve` (krylov.py:60-141) on a CudaGridState: the
  reference's host-side CG with the device cycle as preconditioner --
  histories, iteration counts and the solution bit-identical to the
  reference on its GridState;
* `kcycle.cycle.solve_standalone` (cycle.py:303-366) through a build_state
  shim: bit-identical reports;
* the reference's own test modules test_cycle.py and test_krylov.py, run
  unchanged with `build_state` returning CudaGridState (tests/refshim.py).
"""

import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "kcycle")):
    pytest.skip("reference not installed in baseline/_ref (tools/install_reference.sh)", allow_module_level=True)
if REF not in sys.path:
    sys.path.insert(0, REF)

import kcycle  # noqa: E402  (the reference, from baseline/_ref)
import kcycle.cycle as rc  # noqa: E402
import kcycle.krylov as rk  # noqa: E402
import kcycle.mesh as rm  # noqa: E402
import kcycle.stencil as rs  # noqa: E402

kc = pytest.importorskip("paper_2010_00626_b200")
from paper_2010_00626_b200.cycle import CudaGridState  # noqa: E402

INF = math.inf
assert os.path.dirname(kcycle.__file__).startswith(REF), kcycle.__file__


def cuda_state(problem, cfg):
    """CudaGridState from the reference's own hierarchy objects."""
    spec = rm.build_hierarchy(cfg.n, cfg.coarsening)
    ops = rs.operator_hierarchy(problem, spec, cfg.coarse_op)
    return CudaGridState(spec, ops, cfg.smoother, cfg.nu1, cfg.nu2)


def pair(n, kappa, seed, eps=1e-4, phi=45.0, **kw):
    problem = rs.ProblemSpec(epsilon=eps, phi=phi, seed=seed)
    cfg = rc.CycleConfig(n=n, kappa=kappa, **kw)
    ref = rc.build_state(problem, cfg)
    dev = cuda_state(problem, cfg)
    rng = np.random.default_rng(seed)
    v0, f0 = rng.random(ref.v[0].shape), rng.standard_normal(ref.f[0].shape)
    ref.v[0], ref.f[0] = v0.copy(), f0.copy()
    dev.v[0], dev.f[0] = v0, f0
    return problem, cfg, ref, dev


@pytest.mark.parametrize("n", [5, 7, 9])
@pytest.mark.parametrize("kappa", [1, 2, 3, 4, INF])
def test_reference_run_cycle_drives_cuda_state(n, kappa):
    _, cfg, ref, dev = pair(n, kappa, seed=n)
    for c in range(2):
        s_ref, s_dev = rc.CycleStats.for_levels(n), rc.CycleStats.for_levels(n)
        rc.run_cycle(ref, cfg, s_ref)
        rc.run_cycle(dev, cfg, s_dev)
        assert np.array_equal(dev.v[0], ref.v[0]), (n, kappa, c)
        assert s_dev == s_ref
    # the coarse levels too (every level's v after the cycle)
    for lvl in range(n):
        assert np.array_equal(dev.v[lvl], ref.v[lvl]), lvl
    dev.close()


@pytest.mark.parametrize("form", ["gamma1", "gamma2", "f"])
def test_reference_classical_forms_drive_cuda_state(form):
    n = 7
    _, cfg, ref, dev = pair(n, 1, seed=3)
    for st in (ref, dev):
        stats = rc.CycleStats.for_levels(n)
        if form == "f":
            rc.f_cycle(st, 1, stats)
        else:
            rc.gamma_cycle(st, 1, int(form[-1]), stats)
    assert np.array_equal(dev.v[0], ref.v[0])
    dev.close()


@pytest.mark.parametrize("smoother,coarsening", [("zebra-x", "semi-y"), ("zebra-xy", "full")])
def test_reference_kappa_cycle_zebra_on_cuda_state(smoother, coarsening):
    from kcycle.smoother import SmootherKind, SmootherSpec
    n = 6
    kw = dict(smoother=SmootherSpec(SmootherKind(smoother), 1.0), coarsening=rm.Coarsening(coarsening), nu1=2, nu2=2)
    _, cfg, ref, dev = pair(n, 2, seed=5, eps=1e-3, phi=30.0, **kw)
    for _ in range(2):
        rc.kappa_cycle(ref, 1, 2, rc.CycleStats.for_levels(n))
        rc.kappa_cycle(dev, 1, 2, rc.CycleStats.for_levels(n))
    assert np.array_equal(dev.v[0], ref.v[0])
    dev.close()


@pytest.mark.parametrize("n,kappa,stop", [(5, 1, "error"), (5, 3, "residual"), (7, 2, "error"),
                                          (7, INF, "residual"), (9, 2, "residual")])
def test_reference_pcg_solve_on_cuda_state_bit_exact(n, kappa, stop):
    """krylov.py:60-141 unchanged: host CG vectors, the device cycle as M^-1."""
    problem = rs.ProblemSpec(epsilon=1e-4, phi=45.0, seed=0)
    cfg = rc.CycleConfig(n=n, kappa=kappa)
    pc = rk.PcgConfig(cycle=cfg, target_reduction=1e8, stop=stop)
    m = 2 ** n - 1
    x0 = np.random.default_rng(0).random((m, m))
    f = np.zeros((m, m))
    ref = rk.pcg_solve(rc.build_state(problem, cfg), f, pc, x0=x0)
    dev_state = cuda_state(problem, cfg)
    dev = rk.pcg_solve(dev_state, f, pc, x0=x0)
    assert dev.status == ref.status == "converged"
    assert dev.iterations == ref.iterations
    assert dev.per_cycle_reduction == ref.per_cycle_reduction
    assert dev.final_error_norm == ref.final_error_norm
    assert np.array_equal(dev.solution, ref.solution)
    assert dev.stats.visits == ref.stats.visits and dev.stats.kernel_launches == ref.stats.kernel_launches
    dev_state.close()


@pytest.mark.parametrize("n,kappa", [(6, 1), (7, 3), (8, INF)])
def test_reference_solve_standalone_through_build_state_shim(n, kappa, monkeypatch):
    problem = rs.ProblemSpec(epsilon=1e-4, phi=45.0, seed=0)
    cfg = rc.CycleConfig(n=n, kappa=kappa)
    ref = rc.solve_standalone(problem, cfg, 1e8)
    built = []

    def shim(p, c):
        built.append(cuda_state(p, c))
        return built[-1]

    monkeypatch.setattr(rc, "build_state", shim)
    dev = rc.solve_standalone(problem, cfg, 1e8)
    assert len(built) == 1 and isinstance(built[0], CudaGridState)
    assert (dev.status, dev.iterations) == (ref.status, ref.iterations)
    assert dev.per_cycle_reduction == ref.per_cycle_reduction
    assert dev.final_error_norm == ref.final_error_norm
    assert np.array_equal(dev.solution, ref.solution)
    assert dev.stats == ref.stats


def test_reference_test_modules_pass_on_cuda_state(tmp_path):
    """The reference's own test_cycle.py and test_krylov.py, unchanged, with
    build_state returning CudaGridState (tests/refshim.py)."""
    tdir = os.path.join(REF, "kcycle_tests")
    if not os.path.isdir(tdir):
        pytest.skip("reference tests not copied into baseline/_ref")
    report = tmp_path / "refshim.json"
    env = dict(os.environ, KC_REF_PATH=REF, KC_REPO_ROOT=ROOT, KC_REFSHIM_REPORT=str(report),
               PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "tests"), REF, ROOT]),
               PYTHONDONTWRITEBYTECODE="1", OPENBLAS_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "refshim", "-p", "no:cacheprovider",
           "--rootdir", tdir, "-c", os.devnull,
           os.path.join(tdir, "test_cycle.py"), os.path.join(tdir, "test_krylov.py")]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1200)
    tail = (res.stdout + res.stderr)[-3000:]
    assert res.returncode == 0, tail
    built = json.loads(report.read_text())["cuda_states"]
    assert built >= 10, (built, tail)  # the device path really ran


def _flip_second(n_calls):
    """Identity preconditioner on the first application, -r from the second:
    the r.z_next <= 0 breakdown at iteration 1 (krylov.py:121-123)."""
    calls = []

    def pre(r):
        calls.append(1)
        return r.copy() if len(calls) < n_calls else -r

    return pre


@pytest.mark.parametrize("flip_at", [2, 3])
def test_pcg_rz_breakdown_history_vs_reference(flip_at):
    """An r.z breakdown after a measured step keeps that step's measure:
    the repo's pcg_solve reports the reference's iterations, status, final
    measure and reduction list (the ADVICE round-1 history-length fix)."""
    problem = rs.ProblemSpec(epsilon=1.0, phi=0.0, seed=0)
    cfg = rc.CycleConfig(n=3, kappa=1)
    x0 = np.random.default_rng(0).random((7, 7))
    pc = rk.PcgConfig(cycle=cfg, target_reduction=1e8, stop="error")
    ref = rk.pcg_solve(rc.build_state(problem, cfg), np.zeros((7, 7)), pc, x0=x0, precondition=_flip_second(flip_at))
    mine_state = kc.build_state(kc.ProblemSpec(1.0, 0.0, seed=0), kc.CycleConfig(n=3, kappa=1))
    mine = kc.pcg_solve(mine_state, np.zeros((7, 7)), kc.PcgConfig(cycle=kc.CycleConfig(n=3, kappa=1),
                                                                    target_reduction=1e8, stop="error"),
                        x0=x0, precondition=_flip_second(flip_at))
    assert ref.status == mine.status == "breakdown"
    assert mine.iterations == ref.iterations == flip_at - 1
    assert len(mine.per_cycle_reduction) == len(ref.per_cycle_reduction)
    assert mine.final_error_norm == pytest.approx(ref.final_error_norm, rel=1e-12)
    mine_state.close()


def test_pcg_precondition_exception_surfaces_at_once():
    """A raising user preconditioner stops the device loop at the next
    r.z test (NaN z) and the exception reaches the caller."""
    calls = []

    def bad(r):
        calls.append(1)
        raise RuntimeError("boom")

    st = kc.build_state(kc.ProblemSpec(1.0, 0.0), kc.CycleConfig(n=3, kappa=1))
    with pytest.raises(RuntimeError, match="boom"):
        kc.pcg_solve(st, np.zeros((7, 7)), kc.PcgConfig(cycle=kc.CycleConfig(n=3, kappa=1), stop="error"),
                     x0=np.ones((7, 7)), precondition=bad)
    assert len(calls) == 1
    st.close()


def test_solve_standalone_rejects_mismatched_state():
    """a caller-supplied state must match problem and config."""
    p = kc.ProblemSpec(1e-4, 45.0)
    st = kc.build_state(p, kc.CycleConfig(n=5, kappa=2))
    with pytest.raises(ValueError):
        kc.solve_standalone(p, kc.CycleConfig(n=6, kappa=2), 1e8, state=st)
    with pytest.raises(ValueError):
        kc.solve_standalone(p, kc.CycleConfig(n=5, kappa=2, nu1=1), 1e8, state=st)
    with pytest.raises(ValueError):
        kc.solve_standalone(kc.ProblemSpec(1e-3, 45.0), kc.CycleConfig(n=5, kappa=2), 1e8, state=st)
    rep = kc.solve_standalone(p, kc.CycleConfig(n=5, kappa=3), 1e8, state=st)  # kappa may differ
    assert rep.status == "converged"
    st.close()
