"""Pin the CPU oracle to golden vectors produced by the REAL reference.

tests/golden/make_golden.py ran /root/reference/pkg/src/kcycle in the build
container and stored its outputs; here the oracle restatement must reproduce
them (bit-exact for all elementwise work and whole cycles, ~1 ulp for norms).
"""

import hashlib
import math

import numpy as np
import pytest

from conftest import golden_exists, load_json, load_npz
from oracle import kcycle_oracle as O

INF = math.inf


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def test_stencil_hierarchies_bit_exact(golden_stencils):
    for e in golden_stencils:
        ws = O.hierarchy(e["epsilon"], e["phi"], e["n"], e["coarse_op"])
        got = [[float(x).hex() for x in w.ravel()] for w in ws]
        assert got == e["w_hex"], (e["epsilon"], e["phi"], e["coarse_op"])


def test_tap_drop_rule():
    """ndimage drops |w| <= DBL_EPSILON: a 2.2e-16 tap contributes 0."""
    u = np.ones((3, 3))
    w = np.zeros((3, 3))
    w[0, 0] = np.finfo(float).eps
    assert O.apply(w, u)[1, 1] == 0.0
    w[0, 0] = 2.3e-16
    assert O.apply(w, u)[1, 1] == 2.3e-16


def test_kernels_bit_exact():
    z = load_npz("kernels.npz")
    meta = load_json("kernels_meta.json")
    for key in meta["keys"]:
        u, f, w = z[key + "_u"], z[key + "_f"], z[key + "_w"]
        assert np.array_equal(O.apply(w, u), z[key + "_apply"]), key
        assert np.array_equal(O.residual(w, u, f), z[key + "_residual"]), key
        assert np.array_equal(O.jacobi(w, u, f, 0.8), z[key + "_jacobi"]), key
        assert np.array_equal(O.relax(w, u, f, 0.8, 3), z[key + "_relax3"]), key
        if key + "_restrict" in z:
            assert np.array_equal(O.restrict(f), z[key + "_restrict"]), key
        assert np.array_equal(O.prolong(u), z[key + "_prolong"]), key
        if key + "_coarsest" in z:
            assert np.array_equal(O.coarsest(w, f), z[key + "_coarsest"]), key


@pytest.mark.parametrize("n", [3, 5])
@pytest.mark.parametrize("kname", ["1", "2", "3", "4", "W"])
def test_cycles_random_state_bit_exact(n, kname):
    """random v and f (test_cycle.py:39-46 helper, eps=0.5, phi=30)."""
    z = load_npz("cycles.npz")
    h = O.Hierarchy(O.hierarchy(0.5, 30.0, n))
    key = f"n{n}_k{kname}"
    h.v[0] = z[key + "_v0"].copy()
    h.f[0] = z[key + "_f0"].copy()
    kappa = n if kname == "W" else int(kname)
    for c in range(1, 4):
        h.cycle(kappa)
        assert np.array_equal(h.v[0], z[f"{key}_c{c}"]), (key, c)
    meta = load_json("cycles_meta.json")["random_state"][key]
    assert [sum(1 for t in h.trace if t[0] == l) for l in range(1, n + 1)] == meta["visits"]


@pytest.mark.parametrize("kname", ["1", "2", "4", "W"])
def test_cycles_paper_problem_sha(kname):
    meta = load_json("cycles_meta.json")["paper_problem"][f"n7_k{kname}"]
    n = 7
    h = O.Hierarchy(O.hierarchy(1e-4, 45.0, n))
    h.v[0] = np.random.default_rng(0).random((127, 127))
    kappa = n if kname == "W" else int(kname)
    for c in range(10):
        h.cycle(kappa)
        assert sha(h.v[0]) == meta["sha256"][c], c
        assert O.norm2(h.v[0]) == pytest.approx(meta["norms"][c], rel=1e-14)


@pytest.mark.parametrize("key", ["n5_k1", "n5_k3", "n5_kW", "n7_k1", "n7_k2", "n7_k4"])
def test_standalone_histories(key):
    g = load_json("solves_small.json")["standalone"][key]
    kappa = INF if g["kappa"] == "W" else int(g["kappa"])
    r = O.standalone(g["epsilon"], g["phi"], g["n"], kappa, target=1e10, seed=g["seed"],
                     max_cycles=len(g["err_hist"]) - 1)
    assert r["iterations"] == g["iters_error_1e10"]
    e = np.array(r["err_hist"])
    ge = np.array(g["err_hist"][: len(e)])
    assert np.max(np.abs(e - ge) / ge) < 1e-13
    res = np.array(r["res_hist"])
    gr = np.array(g["res_hist"][: len(res)])
    assert np.max(np.abs(res - gr) / gr) < 1e-13


@pytest.mark.parametrize("key", ["n5_k1", "n5_k2", "n7_k3"])
def test_pcg_counts(key):
    g = load_json("solves_small.json")["pcg"][key]
    kappa = INF if g["kappa"] == "W" else int(g["kappa"])
    for stop, tgt, name in (("error", 1e8, "error_1e8"), ("residual", 1e10, "residual_1e10")):
        r = O.pcg(g["epsilon"], g["phi"], g["n"], kappa, target=tgt, stop=stop, seed=g["seed"])
        assert r["status"] == "converged"
        assert r["iterations"] == g["iters"][name], (stop, tgt)
        ref = np.array(g["x_hist"] if stop == "error" else g["r_hist"])[: len(r["hist"])]
        assert np.max(np.abs(np.array(r["hist"]) - ref) / ref) < 1e-10


def test_level_calls_closed_form():
    d = load_json("dry_stats.json")
    for key, rec in d.items():
        n = int(key.split("_")[0][1:])
        kn = key.split("_")[1][1:]
        kappa = INF if kn == "W" else int(kn)
        assert O.level_calls(kappa, n) == rec["visits"], key


@pytest.mark.skipif(not golden_exists("solve_n12_k4.json"), reason="n=12 golden not generated")
def test_n12_first_cycle_sha():
    """One n=12 cycle (4095^2) of the oracle equals the reference bit-for-bit."""
    g = load_json("solve_n12_k4.json")
    h = O.Hierarchy(O.hierarchy(1e-4, 45.0, 12))
    h.v[0] = np.random.default_rng(0).random((4095, 4095))
    assert O.norm2(h.v[0]) == pytest.approx(g["err_hist"][0], rel=1e-14)
    h.cycle(4)
    assert sha(h.v[0]) == g["sha256"]["1"]


# ---------------------------------------------------------------------------
# zebra line relaxation, y-semi-coarsening, line coarsest solve (§8(f)1)
# ---------------------------------------------------------------------------

def test_gtsv_restatement_matches_scipy_solve_banded():
    """The oracle's dgtsv restatement is bit-identical to scipy's
    solve_banded((1,1)) -- the call inside zebra_line_sweep (smoother.py:133)
    -- with and without row interchanges."""
    import scipy.linalg as sl
    rng = np.random.default_rng(0)
    for trial in range(200):
        n = int(rng.integers(1, 50))
        lo, di, up = rng.standard_normal(3) * (1.0 if trial % 2 else np.array([0.3, 2.0, 0.4]))
        ab = np.zeros((3, n))
        ab[0, 1:], ab[1, :], ab[2, :-1] = up, di, lo
        b = rng.standard_normal((n, 3))
        ref = sl.solve_banded((1, 1), ab, b)
        got = O.gtsv(np.full(n - 1, lo), np.full(n, di), np.full(n - 1, up), b)
        assert np.array_equal(ref, got), trial


def test_zebra_kernels_vs_reference():
    z = load_npz("zebra.npz")
    meta = load_json("zebra_meta.json")
    for key in meta["kernels"]:
        u, f, w = z[key + "_u"], z[key + "_f"], z[key + "_w"]
        assert np.array_equal(O.zebra(w, u, f, "x"), z[key + "_zx"]), key
        assert np.array_equal(O.zebra(w, u, f, "y"), z[key + "_zy"]), key
        assert np.array_equal(O.relax(w, u, f, 0.8, 2, O.ZEBRA_XY), z[key + "_zxy2"]), key
        if key + "_rsemi" in z:
            assert np.array_equal(O.restrict_semi(f), z[key + "_rsemi"]), key
        assert np.array_equal(O.prolong_semi(u), z[key + "_psemi"]), key
        if key + "_coarsest" in z:
            assert np.array_equal(O.coarsest(w, f, O.SEMI_Y), z[key + "_coarsest"]), key


def test_semi_hierarchies_vs_reference():
    for rec in load_json("zebra_meta.json")["hierarchies"]:
        ws = O.hierarchy(rec["epsilon"], rec["phi"], rec["n"], coarsening=O.SEMI_Y)
        for w, ref in zip(ws, rec["w_hex"]):
            assert [float(x).hex() for x in w.ravel()] == ref, (rec["epsilon"], rec["phi"])


def test_zebra_cycles_vs_reference():
    z = load_npz("zebra.npz")
    for key, rec in load_json("zebra_meta.json")["cycles"].items():
        n = rec["n"]
        ws = O.hierarchy(0.5, 30.0, n, coarsening=rec["coarsening"])
        h = O.Hierarchy(ws, smoother=rec["smoother"], coarsening=rec["coarsening"])
        h.v[0], h.f[0] = z[key + "_v0"].copy(), z[key + "_f0"].copy()
        k = O.eff_kappa(O.INF if rec["kappa"] == "W" else int(rec["kappa"]), n)
        for c in (1, 2):
            h.cycle(k)
            assert np.array_equal(h.v[0], z[f"{key}_c{c}"]), (key, c)


def test_zebra_solves_vs_reference():
    for key, rec in load_json("zebra_meta.json")["solves"].items():
        if rec["n"] > 5:
            continue  # n = 7 cases are covered on the GPU
        out = O.standalone(1e-4, 45.0, rec["n"], int(rec["kappa"]), target=1e8, max_cycles=2000,
                           smoother=rec["smoother"], coarsening=rec["coarsening"], track_residual=False)
        assert out["status"] == rec["status"] and out["iterations"] == rec["iterations"], key
        assert out["err_hist"][-1] == pytest.approx(rec["final_error_norm"], rel=1e-12)
