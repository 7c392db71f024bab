"""Small cases, one per kernel family, for compute-sanitizer (
VERDICT r01 item 6).  Each case runs a few ops of one family on the GPU and
checks the result against the oracle, so a sanitizer run also shows the
case did its work.  Usage (tools/sanitize.sh loops over cases and tools):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py bottom_cluster

Families: k_bottom (16-CTA cluster and single CTA), k_pre / k_post
(streaming), k_ctile_pre / k_ctile_post, the per-op grid kernels, k_zebra_*,
k_pcg_*, k_strip_* (fused and per-op strip passes), both arithmetic builds.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2010_00626_b200 as kc  # noqa: E402
from oracle import kcycle_oracle as O  # noqa: E402


def _cycle_case(n, kappa, arith="exact", env=None, cycles=1):
    for k, v in (env or {}).items():
        os.environ[k] = v
    m = 2 ** n - 1
    rng = np.random.default_rng(n + kappa)
    v0, f0 = rng.random((m, m)), rng.standard_normal((m, m))
    cfg = kc.CycleConfig(n=n, kappa=kappa)
    st = kc.build_state(kc.ProblemSpec(1e-4, 45.0), cfg, arith=arith)
    st.v[0], st.f[0] = v0, f0
    for _ in range(cycles):
        kc.run_cycle(st, cfg, kc.CycleStats.for_levels(n))
    got = st.v[0]
    h = O.Hierarchy(O.hierarchy(1e-4, 45.0, n))
    h.v[0], h.f[0] = v0.copy(), f0.copy()
    for _ in range(cycles):
        h.cycle(kappa)
    d = float(np.max(np.abs(got - h.v[0])))
    tol = 0.0 if arith == "exact" else 1e-12 * float(np.max(np.abs(h.v[0])))
    assert d <= tol, d
    st.close()
    return d


def bottom_cluster():  # 16-CTA cluster entering at 127^2 (n = 8: the whole cycle is one bottom launch)
    return _cycle_case(8, 3, env={"KC_BOT_CLUSTER": "1", "KC_BOT_ENTRY": "127"})


def bottom_cluster_255():
    return _cycle_case(9, 2, env={"KC_BOT_CLUSTER": "1", "KC_BOT_ENTRY": "255"})


def bottom_single():  # one CTA entering at 63^2
    return _cycle_case(7, 3, env={"KC_BOT_CLUSTER": "0"})


def stream():  # k_pre / k_post on 2047^2 and 1023^2 (+ ctiles and bottom below)
    return _cycle_case(11, 2)


def stream_fast():
    return _cycle_case(11, 2, arith="fast")


def ctile():  # column-tile passes on 511^2 .. 127^2 under the streaming levels
    return _cycle_case(10, 3)


def per_op():  # the drop-in per-op kernels (k_jacobi, k_resid_restrict, k_prolong_add, k_coarsest)
    n, kappa = 8, 2
    m = 2 ** n - 1
    rng = np.random.default_rng(5)
    v0, f0 = rng.random((m, m)), rng.standard_normal((m, m))
    st = kc.build_state(kc.ProblemSpec(1e-4, 45.0), kc.CycleConfig(n=n, kappa=kappa))
    st.v[0], st.f[0] = v0, f0
    kc.kappa_cycle(st, 1, kappa, kc.CycleStats.for_levels(n))
    h = O.Hierarchy(O.hierarchy(1e-4, 45.0, n))
    h.v[0], h.f[0] = v0.copy(), f0.copy()
    h.cycle(kappa)
    assert np.array_equal(st.v[0], h.v[0])
    st.close()


def zebra():
    from paper_2010_00626_b200.mesh import Coarsening
    from paper_2010_00626_b200.smoother import SmootherKind, SmootherSpec
    for sm, co in ((SmootherKind.ZEBRA_X, Coarsening.SEMI_Y), (SmootherKind.ZEBRA_ALTERNATING, Coarsening.FULL_STANDARD)):
        cfg = kc.CycleConfig(n=6, kappa=2, smoother=SmootherSpec(sm, 1.0), coarsening=co)
        st = kc.build_state(kc.ProblemSpec(1e-3, 30.0), cfg)
        rng = np.random.default_rng(1)
        st.v[0] = rng.random(st.v[0].shape)
        kc.run_cycle(st, cfg, kc.CycleStats.for_levels(6))
        assert np.all(np.isfinite(st.v[0]))
        st.close()


def pcg():
    n, kappa = 9, 2
    m = 2 ** n - 1
    cfg = kc.CycleConfig(n=n, kappa=kappa)
    st = kc.build_state(kc.ProblemSpec(1e-4, 45.0, seed=0), cfg)
    x0 = np.random.default_rng(0).random((m, m))
    rep = kc.pcg_solve(st, np.zeros((m, m)), kc.PcgConfig(cycle=cfg, target_reduction=1e8, stop="error",
                                                           max_iterations=5), x0=x0)
    assert rep.iterations == 5
    st.close()


def strip():  # fused and per-op strip passes, thread ranks on one GPU
    import threading

    from paper_2010_00626_b200.distributed import DistributedKappaSolver, ThreadComm
    n, world = 9, 2
    m = 2 ** n - 1
    rng = np.random.default_rng(3)
    v0, f0 = rng.random((m, m)), rng.standard_normal((m, m))
    comms = ThreadComm.group(world)
    out = [None] * world
    errs = []

    def run(r):
        try:
            s = DistributedKappaSolver(kc.ProblemSpec(1e-4, 45.0), kc.CycleConfig(n=n, kappa=2), comms[r], min_rows=32)
            s.set_level1("v", v0)
            s.set_level1("f", f0)
            s.cycle()
            out[r] = s.gather_level1()
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    h = O.Hierarchy(O.hierarchy(1e-4, 45.0, n))
    h.v[0], h.f[0] = v0.copy(), f0.copy()
    h.cycle(2)
    assert np.array_equal(out[0], h.v[0])


CASES = {f.__name__: f for f in (bottom_cluster, bottom_cluster_255, bottom_single, stream, stream_fast, ctile,
                                 per_op, zebra, pcg, strip)}

if __name__ == "__main__":
    name = sys.argv[1]
    r = CASES[name]()
    print(f"case {name} ok" + ("" if r is None else f" (max |d| {r:.3g})"))
