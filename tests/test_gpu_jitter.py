"""Race testing of the cluster bottom kernel by schedule perturbation.

compute-sanitizer (racecheck / synccheck) is closed on this GPU pool, so the
bottom kernel -- shared-memory phases, DSMEM halo pushes and broadcasts,
cluster barriers, frame operators, deep-halo strips -- is also built with
KC_BOT_JITTER (libkcb200_jitter.so, libkcb200_fast_jitter.so): about one
warp in four sleeps up to 2 us after every barrier, so a stage that reads
data another warp or CTA has not finished writing would see it and change
the result.  Bar: with jitter, the exact build's cycles stay bit-identical to
the oracle (the reference's arithmetic) and the fast build's stay
bit-identical to the same build without jitter, over repeated runs and the
launch shapes the engine uses (16-CTA cluster with deep halos on the 127^2
entry and 63^2 strips (PH_FRAME127), on the 63^2 strips only (PH_FRAME63),
without, and one CTA).
"""

import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

kc = pytest.importorskip("paper_2010_00626_b200")
from paper_2010_00626_b200 import CycleConfig, CycleStats, ProblemSpec, build_state, run_cycle  # noqa: E402
from oracle import kcycle_oracle as O  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2010_00626_b200")

CHILD = r'''
import hashlib, json, os, sys
import numpy as np
sys.path.insert(0, os.environ["KC_ROOT"])
import paper_2010_00626_b200 as kc
cases = json.loads(sys.argv[1])
out = {}
for c in cases:
    for k, v in c.get("env", {}).items():
        os.environ[k] = v
    n, kap, arith = c["n"], c["kappa"], c["arith"]
    m = 2 ** n - 1
    rng = np.random.default_rng(c["seed"])
    v0, f0 = rng.random((m, m)), rng.standard_normal((m, m))
    cfg = kc.CycleConfig(n=n, kappa=kap)
    shas = []
    for rep in range(c["reps"]):
        st = kc.build_state(kc.ProblemSpec(1e-4, 45.0), cfg, arith=arith)
        st.v[0], st.f[0] = v0, f0
        for _ in range(c["cycles"]):
            kc.run_cycle(st, cfg, kc.CycleStats.for_levels(n))
        shas.append(hashlib.sha256(np.ascontiguousarray(st.v[0]).tobytes()).hexdigest())
        st.close()
    if c.get("time"):
        st = kc.build_state(kc.ProblemSpec(1e-4, 45.0), cfg, arith=arith)
        st.v[0], st.f[0] = v0, f0
        st.run_cycles(kap, 2)
        out[c["name"] + ":ms"] = st.time_cycles(kap, 10) / 10
        st.close()
    for k in c.get("env", {}):
        os.environ.pop(k, None)
    out[c["name"]] = shas
print("JSON" + json.dumps(out))
'''


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _run_jitter(cases):
    env = dict(os.environ, KC_ROOT=ROOT, KCB200_LIB=os.path.join(PKG, "libkcb200_jitter.so"),
               KCB200_LIB_FAST=os.path.join(PKG, "libkcb200_fast_jitter.so"))
    res = subprocess.run([sys.executable, "-c", CHILD, json.dumps(cases)], env=env, capture_output=True, text=True,
                         timeout=1200)
    assert res.returncode == 0, res.stderr[-3000:]
    line = [ln for ln in res.stdout.splitlines() if ln.startswith("JSON")][-1]
    return json.loads(line[4:])


def _cases(arith, shapes, ns, kappas, reps=3, cycles=2):
    out = []
    for shape, env in shapes:
        for n in ns:
            for kap in kappas:
                out.append({"name": f"{arith}-{shape}-n{n}-k{kap}", "n": n, "kappa": kap, "arith": arith,
                            "seed": 100 + n + kap, "reps": reps, "cycles": cycles, "env": env})
    return out


# "barriers": the st.async phases (frame-operator outputs, the 63^2 -> 31^2
# broadcast; mbarrier completion) switched back to DSMEM stores + cluster
# barriers -- a runtime switch of the jitter builds only (kc_bottom.cuh
# KC_ASYNC_ON): the same iterates either way, under perturbation
SHAPES = [("deep", {}), ("deep63", {"KC_DEEP127": "0"}), ("nodeep", {"KC_DEEP": "0"}),
          ("onecta", {"KC_BOT_CLUSTER": "0"}), ("barriers", {"KC_MV_ASYNC": "0", "KC_RB_ASYNC": "0"})]


def test_jitter_libraries_present_and_perturbing():
    """The jitter builds exist and really sleep: the same cycle runs clearly
    slower than in the normal build."""
    for name in ("libkcb200_jitter.so", "libkcb200_fast_jitter.so"):
        assert os.path.exists(os.path.join(PKG, name)), name
    case = {"name": "timing", "n": 9, "kappa": 3, "arith": "exact", "seed": 1, "reps": 1, "cycles": 1, "env": {},
            "time": True}
    got = _run_jitter([case])
    m = 2 ** 9 - 1
    rng = np.random.default_rng(1)
    cfg = CycleConfig(n=9, kappa=3)
    st = build_state(ProblemSpec(1e-4, 45.0), cfg)
    st.v[0], st.f[0] = rng.random((m, m)), rng.standard_normal((m, m))
    st.run_cycles(3, 2)
    plain = st.time_cycles(3, 10) / 10
    st.close()
    assert got["timing:ms"] > 1.2 * plain, (got["timing:ms"], plain)


def test_exact_build_under_jitter_bit_exact_vs_oracle():
    cases = _cases("exact", SHAPES, [8, 9], [1, 2, 3, 9])
    got = _run_jitter(cases)
    for c in cases:
        n, kap = c["n"], c["kappa"]
        m = 2 ** n - 1
        rng = np.random.default_rng(c["seed"])
        v0, f0 = rng.random((m, m)), rng.standard_normal((m, m))
        h = O.Hierarchy(O.hierarchy(1e-4, 45.0, n))
        h.v[0], h.f[0] = v0.copy(), f0.copy()
        for _ in range(c["cycles"]):
            h.cycle(min(kap, n))
        ref = _sha(h.v[0])
        assert got[c["name"]] == [ref] * c["reps"], c["name"]


def test_fast_build_under_jitter_equals_fast_build():
    cases = _cases("fast", SHAPES[:3] + SHAPES[4:], [9, 12], [1, 2, 3, 12], reps=2)
    cases = [c for c in cases if not (c["n"] == 9 and c["kappa"] == 12)]
    got = _run_jitter(cases)
    for c in cases:
        n, kap = c["n"], c["kappa"]
        m = 2 ** n - 1
        rng = np.random.default_rng(c["seed"])
        v0, f0 = rng.random((m, m)), rng.standard_normal((m, m))
        for k, v in c["env"].items():
            os.environ[k] = v
        try:
            cfg = CycleConfig(n=n, kappa=kap)
            st = build_state(ProblemSpec(1e-4, 45.0), cfg, arith="fast")
            st.v[0], st.f[0] = v0, f0
            for _ in range(c["cycles"]):
                run_cycle(st, cfg, CycleStats.for_levels(n))
            ref = _sha(st.v[0])
            st.close()
        finally:
            for k in c["env"]:
                os.environ.pop(k, None)
        assert got[c["name"]] == [ref] * c["reps"], c["name"]
