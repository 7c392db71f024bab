"""Generate golden fixtures by running the REAL reference package `kcycle`.

Test infrastructure only: this script imports the reference from
/root/reference/pkg/src (present in the build container, absent on the GPU
box) and writes small JSON/NPZ fixtures under tests/golden/ that the oracle
and the GPU parity tests are pinned against.  Nothing in the product path
reads /root/reference.

Usage (run with OPENBLAS_NUM_THREADS=1 so ddot-based norms are the
single-thread values):

    python tests/golden/make_golden.py small
    python tests/golden/make_golden.py solve --n 12 --kappa 4    # long
    python tests/golden/make_golden.py pcg   --n 12 --kappa 4    # long

Every fixture records the reference call it came from:
  * kernels: stencil.apply / residual (stencil.py:108-120),
    smoother.damped_jacobi_sweep (smoother.py:95-100),
    transfer.restrict / prolong (transfer.py:46-87),
    cycle.coarsest_solve (cycle.py:182-190),
    stencil.operator_hierarchy (stencil.py:151-176);
  * cycles: cycle.run_cycle on GridState (cycle.py:144-263);
  * solves: the solve_standalone loop (cycle.py:303-366) and the pcg_solve
    loop (krylov.py:60-141), re-driven step by step so that per-cycle error
    AND true-residual histories can be recorded.  `small` cross-checks the
    re-driven loops against the reference's own solve_standalone / pcg_solve
    reports (iterations and per-cycle reductions identical).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import numpy as np  # noqa: E402

import kcycle  # noqa: E402
from kcycle import cycle as kc  # noqa: E402
from kcycle import krylov as kk  # noqa: E402
from kcycle import mesh as km  # noqa: E402
from kcycle import smoother as ksm  # noqa: E402
from kcycle import stencil as kst  # noqa: E402
from kcycle import transfer as ktr  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
INF = math.inf
KAPPAS = (1, 2, 3, 4, INF)


def kname(kappa) -> str:
    return "W" if kappa == INF else str(int(kappa))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def dump(name: str, obj) -> None:
    path = os.path.join(HERE, name)
    tmp = path + ".tmp"
    with open(tmp, "w") as fh:
        json.dump(obj, fh, indent=1)
    os.replace(tmp, path)


def problem_config(n, kappa, eps=1e-4, phi=45.0, seed=0, **kw):
    problem = kst.ProblemSpec(epsilon=eps, phi=phi, seed=seed)
    config = kc.CycleConfig(n=n, kappa=kappa, **kw)
    return problem, config


# ----------------------------------------------------------------------------
# small fixtures
# ----------------------------------------------------------------------------

STENCIL_CASES = [(1e-4, 45.0), (0.1, 45.0), (1.0, 0.0), (0.5, 30.0), (1e-3, 45.0), (0.2, 30.0)]


def gen_stencils():
    out = []
    for eps, phi in STENCIL_CASES:
        for coarse_op in ("galerkin", "rediscretize"):
            spec = km.build_hierarchy(14, km.Coarsening.FULL_STANDARD)
            ops = kst.operator_hierarchy(kst.ProblemSpec(epsilon=eps, phi=phi), spec, coarse_op)
            out.append({
                "epsilon": eps, "phi": phi, "coarse_op": coarse_op, "n": 14,
                "w": [op.w.ravel().tolist() for op in ops],
                "w_hex": [[float(x).hex() for x in op.w.ravel()] for op in ops],
            })
    dump("stencils.json", out)


def gen_kernels():
    """Per-kernel KATs on random data: bit-exact reference outputs."""
    rng = np.random.default_rng(2010_00626)
    arrays = {}
    meta = []
    ops = kst.operator_hierarchy(kst.ProblemSpec(1e-4, 45.0),
                                 km.build_hierarchy(7, km.Coarsening.FULL_STANDARD))
    for side in (1, 3, 7, 15, 31, 63):
        for li, op in ((0, ops[0]), (3, ops[3])):
            key = f"s{side}_l{li}"
            u = rng.random((side, side))
            f = rng.standard_normal((side, side))
            arrays[key + "_u"] = u
            arrays[key + "_f"] = f
            arrays[key + "_w"] = op.w
            arrays[key + "_apply"] = kst.apply(op, u)
            arrays[key + "_residual"] = kst.residual(op, u, f)
            arrays[key + "_jacobi"] = ksm.damped_jacobi_sweep(op, u, f, 0.8)
            arrays[key + "_relax3"] = ksm.relax(op, u, f, ksm.SmootherSpec(ksm.SmootherKind.DAMPED_JACOBI, 0.8), 3)
            if side >= 3:
                arrays[key + "_restrict"] = ktr.restrict(f, km.Coarsening.FULL_STANDARD)
            arrays[key + "_prolong"] = ktr.prolong(u, km.Coarsening.FULL_STANDARD)
            if side == 1:
                arrays[key + "_coarsest"] = kc.coarsest_solve(op, f, km.Coarsening.FULL_STANDARD)
            meta.append(key)
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **arrays)
    dump("kernels_meta.json", {"keys": meta, "omega": 0.8,
                               "source": "kcycle stencil/smoother/transfer/cycle, see make_golden.py"})


def random_state(n, seed=7, eps=0.5, phi=30.0, **kw):
    """Mirror of the reference test helper test_cycle.py:39-46."""
    problem = kst.ProblemSpec(epsilon=eps, phi=phi)
    config = kc.CycleConfig(n=n, kappa=1, **kw)
    state = kc.build_state(problem, config)
    rng = np.random.default_rng(seed)
    state.v[0] = rng.random(state.v[0].shape)
    state.f[0] = rng.random(state.f[0].shape)
    return state


def gen_cycles():
    """Iterates after consecutive cycles, random v AND f (all levels touched)."""
    arrays = {}
    meta = {}
    for n in (3, 5):
        for kappa in (1, 2, 3, 4, INF):
            state = random_state(n)
            cfg = kc.CycleConfig(n=n, kappa=kappa)
            stats = kc.CycleStats.for_levels(n)
            arrays[f"n{n}_k{kname(kappa)}_v0"] = state.v[0].copy()
            arrays[f"n{n}_k{kname(kappa)}_f0"] = state.f[0].copy()
            for c in range(1, 4):
                kc.run_cycle(state, cfg, stats)
                arrays[f"n{n}_k{kname(kappa)}_c{c}"] = state.v[0].copy()
            meta[f"n{n}_k{kname(kappa)}"] = {"visits": stats.visits,
                                              "kernel_launches": stats.kernel_launches,
                                              "unknown_touches": stats.unknown_touches}
    np.savez_compressed(os.path.join(HERE, "cycles.npz"), **arrays)
    # n = 7 and 9 paper problem: sha256 of the iterate after each of 10 cycles
    hashes = {}
    for n in (7, 9):
        for kappa in KAPPAS:
            problem, cfg = problem_config(n, kappa)
            state = kc.build_state(problem, cfg)
            state.v[0] = np.random.default_rng(0).random(state.v[0].shape)
            stats = kc.CycleStats.for_levels(n)
            hs, norms = [], []
            for _ in range(10):
                kc.run_cycle(state, cfg, stats)
                hs.append(sha(state.v[0]))
                norms.append(km.norm2(state.v[0]))
            hashes[f"n{n}_k{kname(kappa)}"] = {"sha256": hs, "norms": norms}
    dump("cycles_meta.json", {"random_state": meta, "paper_problem": hashes})


def track_standalone(n, kappa, err_target=1e10, res_target=1e10, cap=20000,
                     out_name=None, eps=1e-4, phi=45.0, seed=0, sha_at=(1, 2, 5, 10, 20, 50, 100)):
    """Re-driven solve_standalone loop (cycle.py:320-353) recording per-cycle
    error norm ||v_k|| and true residual norm ||f - A v_k|| (f = 0)."""
    problem, cfg = problem_config(n, kappa, eps=eps, phi=phi, seed=seed)
    state = kc.build_state(problem, cfg)
    ny, nx = state.v[0].shape
    state.v[0] = np.random.default_rng(problem.seed).random((ny, nx))
    a0 = state.ops[0]
    stats = kc.CycleStats.for_levels(n)
    e0 = km.norm2(state.v[0])
    r0 = km.norm2(kst.residual(a0, state.v[0], state.f[0]))
    err, res = [e0], [r0]
    hashes = {}
    it_err = it_res = it_e8 = None
    t_cycles = 0.0
    rec = {}

    def snapshot(done):
        rec.update({
            "n": n, "kappa": kname(kappa), "epsilon": eps, "phi": phi, "seed": seed,
            "omega": 0.8, "nu1": 2, "nu2": 2, "coarsening": "full", "coarse_op": "galerkin",
            "err_hist": err, "res_hist": res, "sha256": hashes,
            "iters_error_1e8": it_e8, "iters_error_1e10": it_err, "iters_residual_1e10": it_res,
            "cycle_seconds_mean": t_cycles / max(1, len(err) - 1),
            "complete": done, "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
        })
        if out_name:
            dump(out_name, rec)

    for k in range(1, cap + 1):
        t0 = time.perf_counter()
        kc.run_cycle(state, cfg, stats)
        t_cycles += time.perf_counter() - t0
        e = km.norm2(state.v[0])
        r = km.norm2(kst.residual(a0, state.v[0], state.f[0]))
        err.append(e)
        res.append(r)
        if k in sha_at:
            hashes[str(k)] = sha(state.v[0])
        if it_e8 is None and e <= e0 / 1e8:
            it_e8 = k
            hashes[str(k)] = sha(state.v[0])
        if it_err is None and e <= e0 / err_target:
            it_err = k
            hashes[str(k)] = sha(state.v[0])
        if it_res is None and r <= r0 / res_target:
            it_res = k
            hashes[str(k)] = sha(state.v[0])
        if it_err is not None and it_res is not None:
            break
        if out_name and k % 25 == 0:
            snapshot(False)
    snapshot(True)
    return rec


def track_pcg(n, kappa, cap=5000, out_name=None, eps=1e-4, phi=45.0, seed=0):
    """Re-driven pcg_solve loop (krylov.py:74-128) with f = 0 and
    x0 = default_rng(seed).random (the CLI setup, cli.py:174-180), recording
    per-iteration ||x|| (stop="error"), recursive ||r|| (stop="residual") and
    the true residual ||f - A x||."""
    problem, cfg = problem_config(n, kappa, eps=eps, phi=phi, seed=seed)
    state = kc.build_state(problem, cfg)
    x0 = np.random.default_rng(seed).random(state.v[0].shape)
    f = np.zeros_like(x0)
    a0 = state.ops[0]
    stats = kc.CycleStats.for_levels(n)
    x = x0.astype(float).copy()
    r = f - kst.apply(a0, x)

    def precondition(res):
        state.zero_guess(1)
        state.f[0] = res.copy()
        kc.run_cycle(state, cfg, stats)
        return state.v[0].copy()

    xs = [km.norm2(x)]
    rs = [km.norm2(r)]
    ts = [km.norm2(f - kst.apply(a0, x))]
    rz_hist, pap_hist = [], []
    status = "max_cycles"
    z = precondition(r)
    rz = km.dot(r, z)
    rz_hist.append(rz)
    it = {"error_1e8": None, "error_1e10": None, "residual_1e8": None, "residual_1e10": None,
          "true_residual_1e10": None}
    rec = {}
    t_it = 0.0

    def snapshot(done):
        rec.update({"n": n, "kappa": kname(kappa), "epsilon": eps, "phi": phi, "seed": seed,
                    "x_hist": xs, "r_hist": rs, "true_res_hist": ts, "rz_hist": rz_hist,
                    "pap_hist": pap_hist, "iters": it, "status": status, "complete": done,
                    "iteration_seconds_mean": t_it / max(1, len(xs) - 1)})
        if out_name:
            dump(out_name, rec)

    if rz <= 0.0:
        status = "breakdown"
    else:
        p = z
        for k in range(1, cap + 1):
            t0 = time.perf_counter()
            ap = kst.apply(a0, p)
            pap = km.dot(p, ap)
            pap_hist.append(pap)
            if pap <= 0.0:
                status = "breakdown"
                break
            alpha = rz / pap
            x += alpha * p
            r -= alpha * ap
            xs.append(km.norm2(x))
            rs.append(km.norm2(r))
            ts.append(km.norm2(f - kst.apply(a0, x)))
            for key, hist, tgt in (("error_1e8", xs, 1e8), ("error_1e10", xs, 1e10),
                                   ("residual_1e8", rs, 1e8), ("residual_1e10", rs, 1e10),
                                   ("true_residual_1e10", ts, 1e10)):
                if it[key] is None and hist[-1] <= hist[0] / tgt:
                    it[key] = k
            if all(v is not None for v in it.values()):
                status = "converged"
                t_it += time.perf_counter() - t0
                break
            z = precondition(r)
            rz_next = km.dot(r, z)
            rz_hist.append(rz_next)
            if rz_next <= 0.0:
                status = "breakdown"
                break
            p = z + (rz_next / rz) * p
            rz = rz_next
            t_it += time.perf_counter() - t0
            if out_name and k % 10 == 0:
                snapshot(False)
    snapshot(True)
    return rec


def gen_solves_small():
    out = {"standalone": {}, "pcg": {}}
    for n in (5, 7, 9):
        for kappa in KAPPAS:
            rec = track_standalone(n, kappa, cap=5000)
            # cross-check the re-driven loop against the reference's own driver
            problem, cfg = problem_config(n, kappa)
            rep = kc.solve_standalone(problem, cfg, 1e10, max_cycles=5000)
            assert rep.iterations == rec["iters_error_1e10"], (n, kappa)
            assert rep.final_error_norm == rec["err_hist"][rep.iterations]
            assert rep.per_cycle_reduction == [
                rec["err_hist"][i] / rec["err_hist"][i - 1] for i in range(1, rep.iterations + 1)]
            rep8 = kc.solve_standalone(problem, cfg, 1e8, max_cycles=5000)
            assert rep8.iterations == rec["iters_error_1e8"]
            rec["reference_report_1e10"] = {"status": rep.status, "iterations": rep.iterations,
                                            "final_error_norm": rep.final_error_norm,
                                            "asymptotic_factor": rep.asymptotic_factor,
                                            "kernel_launches": rep.stats.kernel_launches,
                                            "unknown_touches": rep.stats.unknown_touches,
                                            "visits": rep.stats.visits}
            if n == 9:  # keep n=9 fixtures small: counts and norms only at coarse stride
                rec["sha256"] = {}
            out["standalone"][f"n{n}_k{kname(kappa)}"] = rec
            prec = track_pcg(n, kappa)
            for stop, tgt, key in (("error", 1e8, "error_1e8"), ("error", 1e10, "error_1e10"),
                                   ("residual", 1e10, "residual_1e10")):
                state = kc.build_state(problem, cfg)
                x0 = np.random.default_rng(0).random(state.v[0].shape)
                pr = kk.pcg_solve(state, np.zeros_like(x0),
                                  kk.PcgConfig(cycle=cfg, target_reduction=tgt, stop=stop), x0=x0)
                assert pr.iterations == prec["iters"][key], (n, kappa, key, pr.iterations, prec["iters"])
                prec.setdefault("reference_reports", {})[key] = {
                    "status": pr.status, "iterations": pr.iterations,
                    "final_error_norm": pr.final_error_norm,
                    "visits": pr.stats.visits}
            out["pcg"][f"n{n}_k{kname(kappa)}"] = prec
            print(f"n={n} kappa={kname(kappa)}: standalone {rec['iters_error_1e10']}/"
                  f"{rec['iters_residual_1e10']} pcg {prec['iters']}", flush=True)
    # Poisson sanity and a second seed/angle
    out["standalone"]["poisson_n7_k1"] = track_standalone(7, 1, eps=1.0, phi=0.0, cap=200)
    out["standalone"]["n6_k2_eps0.1_phi30_seed3"] = track_standalone(6, 2, eps=0.1, phi=30.0, seed=3, cap=2000)
    dump("solves_small.json", out)


def gen_dry():
    """CycleStats of DryState-driven cycles (cycle.py:114-141)."""
    out = {}
    for n in (1, 2, 3, 5, 7, 12, 14):
        for kappa in (1, 2, 3, 4, 5, INF):
            for nu1, nu2 in ((2, 2), (1, 1), (0, 0), (1, 2)):
                st = kc.CycleStats.for_levels(n)
                kc.run_cycle(kc.DryState(n, nu1, nu2), kc.CycleConfig(n=n, kappa=kappa, nu1=nu1, nu2=nu2), st)
                key = f"n{n}_k{kname(kappa)}_nu{nu1}{nu2}"
                rec = {"visits": st.visits, "kernel_launches": st.kernel_launches,
                       "unknown_touches": st.unknown_touches, "trace_len": len(st.trace)}
                if len(st.trace) <= 200:
                    rec["trace"] = st.trace
                out[key] = rec
    dump("dry_stats.json", out)


def gen_costmodel():
    """Closed forms, model predictions, fits and turning points (costmodel.py)."""
    from kcycle import costmodel as cm
    out = {"cells": [], "f_factor": [], "n_ops": [], "turning_points": [], "fit": None}
    for kappa in (1, 2, 3, 4, 5, 6, INF):
        for n in range(1, 15):
            cell = {"kappa": kname(kappa), "n": n,
                    "level_calls": [cm.level_calls(kappa, l) for l in range(1, n + 1)],
                    "total_calls": cm.total_calls(kappa, n),
                    "n_gpu_calls": {str(nu): cm.n_gpu_calls(kappa, n, nu) for nu in (0, 2, 4)},
                    "ops_per_unknown": cm.ops_per_unknown(kappa),
                    "predicted_ms_paper": cm.predict_runtime(cm.CostModelParams(2.48e-3, 1.18e-6, 4), kappa, n)}
            if kappa != INF:
                cell["histogram"] = {str(k): v for k, v in cm.coarse_counter_histogram(kappa, n).items()}
            out["cells"].append(cell)
    for kappa in (1, 2, 3, 7, INF):
        for c in (0.2, 0.25, 0.3, 0.45, 0.5):
            try:
                v = cm.f_factor(kappa, c)
            except ValueError:
                v = None
            out["f_factor"].append({"kappa": kname(kappa), "c": c, "value": v})
    spec = cm.OpCountSpec(C=1.3, Ctilde=2.7, N1=1.0)
    for kappa in (1, 2, 3, 5, INF):
        for c in (0.2, 0.25, 0.3):
            for n in (1, 3, 7, 12):
                out["n_ops"].append({"kappa": kname(kappa), "c": c, "n": n, "value": cm.n_ops_model(kappa, c, n, spec)})
    for kappa in (1, 2, 3, 4, INF):
        tp = cm.turning_point(cm.CostModelParams(2.48e-3, 1.18e-6, 4), kappa)
        out["turning_points"].append({"kappa": kname(kappa), "n_tp": tp.n_tp, "N_tp": tp.N_tp, "converged": tp.converged})
    rows = [(k, n, 0.01 * cm.n_gpu_calls(k, n, 4) + 3e-7 * (2 ** n - 1) ** 2 * cm.ops_per_unknown(k) * (1 + 0.01 * ((n * 7 + int(k if k != INF else 9)) % 5 - 2)))
            for k in (1, 2, 3, 4, INF) for n in range(4, 14)]
    a, b = cm.fit_params(rows, nu=4)
    out["fit"] = {"rows": [[kname(k), n, t] for k, n, t in rows], "alpha": a, "beta": b}
    dump("costmodel.json", out)


ZEBRA_CONFIGS = [  # (smoother, coarsening) pairs of the paper's solvers 3-6
    ("zebra-xy", "full"), ("zebra-x", "semi-y"), ("zebra-y", "full"), ("jacobi", "semi-y"), ("zebra-x", "full"),
]
_SK = {"jacobi": None, "zebra-x": "ZEBRA_X", "zebra-y": "ZEBRA_Y", "zebra-xy": "ZEBRA_ALTERNATING"}


def _smoother(name):
    return ksm.SmootherSpec(ksm.SmootherKind.DAMPED_JACOBI if name == "jacobi" else getattr(ksm.SmootherKind, _SK[name]),
                            0.8)


def _coarsening(name):
    return km.Coarsening.FULL_STANDARD if name == "full" else km.Coarsening.SEMI_Y


def gen_zebra():
    """Zebra line relaxation, y-semi-coarsening and the line coarsest solve
    (smoother.py:71-163, transfer.py:46-87, cycle.py:182-200): kernel KATs,
    semi-y Galerkin hierarchies, cycle iterates and small solves."""
    rng = np.random.default_rng(4)
    arrays, meta = {}, {"kernels": [], "cycles": {}, "solves": {}, "hierarchies": []}
    full = kst.operator_hierarchy(kst.ProblemSpec(1e-4, 45.0), km.build_hierarchy(6, km.Coarsening.FULL_STANDARD))
    semi = kst.operator_hierarchy(kst.ProblemSpec(1e-4, 45.0), km.build_hierarchy(6, km.Coarsening.SEMI_Y))
    pivot = kst.Stencil9(np.array([[0.1, -0.3, 0.05], [2.5, 0.7, -1.9], [0.2, 0.4, -0.1]]))  # forces row interchanges
    for ny, nx in ((1, 1), (1, 7), (3, 3), (7, 7), (15, 7), (7, 31), (31, 31)):
        for tag, op in (("f0", full[0]), ("f3", full[3]), ("s2", semi[2]), ("piv", pivot)):
            key = f"z{ny}x{nx}_{tag}"
            u = rng.random((ny, nx))
            f = rng.standard_normal((ny, nx))
            arrays[key + "_u"], arrays[key + "_f"], arrays[key + "_w"] = u, f, op.w
            arrays[key + "_zx"] = ksm.zebra_line_sweep(op, u, f, "x")
            arrays[key + "_zy"] = ksm.zebra_line_sweep(op, u, f, "y")
            arrays[key + "_zxy2"] = ksm.relax(op, u, f, ksm.SmootherSpec(ksm.SmootherKind.ZEBRA_ALTERNATING), 2)
            if ny >= 3:
                arrays[key + "_rsemi"] = ktr.restrict(f, km.Coarsening.SEMI_Y)
            arrays[key + "_psemi"] = ktr.prolong(u, km.Coarsening.SEMI_Y)
            if ny == 1 and tag != "piv":
                arrays[key + "_coarsest"] = kc.coarsest_solve(op, f, km.Coarsening.SEMI_Y)
            meta["kernels"].append(key)
    for eps, phi in STENCIL_CASES:
        ops = kst.operator_hierarchy(kst.ProblemSpec(epsilon=eps, phi=phi), km.build_hierarchy(12, km.Coarsening.SEMI_Y))
        meta["hierarchies"].append({"epsilon": eps, "phi": phi, "n": 12,
                                    "w_hex": [[float(x).hex() for x in op.w.ravel()] for op in ops]})
    for sm, co in ZEBRA_CONFIGS:
        for n in (3, 5):
            for kappa in (1, 2, INF):
                problem = kst.ProblemSpec(epsilon=0.5, phi=30.0)
                cfg = kc.CycleConfig(n=n, kappa=kappa, smoother=_smoother(sm), coarsening=_coarsening(co))
                state = kc.build_state(problem, cfg)
                r2 = np.random.default_rng(7 + n)
                state.v[0] = r2.random(state.v[0].shape)
                state.f[0] = r2.random(state.f[0].shape)
                key = f"{sm}_{co}_n{n}_k{kname(kappa)}"
                arrays[key + "_v0"], arrays[key + "_f0"] = state.v[0].copy(), state.f[0].copy()
                stats = kc.CycleStats.for_levels(n)
                for c in range(1, 3):
                    kc.run_cycle(state, cfg, stats)
                    arrays[f"{key}_c{c}"] = state.v[0].copy()
                meta["cycles"][key] = {"smoother": sm, "coarsening": co, "n": n, "kappa": kname(kappa),
                                       "visits": stats.visits, "kernel_launches": stats.kernel_launches,
                                       "unknown_touches": stats.unknown_touches}
        for n in (5, 7):
            for kappa in (1, 2):
                problem, cfg = problem_config(n, kappa, smoother=_smoother(sm), coarsening=_coarsening(co))
                rep = kc.solve_standalone(problem, cfg, 1e8, max_cycles=2000)
                h = [1.0]
                for red in rep.per_cycle_reduction:
                    h.append(h[-1] * red)
                meta["solves"][f"{sm}_{co}_n{n}_k{kname(kappa)}"] = {
                    "smoother": sm, "coarsening": co, "n": n, "kappa": kname(kappa), "status": rep.status,
                    "iterations": rep.iterations, "initial_error_norm": rep.initial_error_norm,
                    "final_error_norm": rep.final_error_norm, "per_cycle_reduction": rep.per_cycle_reduction,
                    "kernel_launches": rep.stats.kernel_launches, "unknown_touches": rep.stats.unknown_touches}
                print(sm, co, n, kname(kappa), rep.status, rep.iterations, flush=True)
    np.savez_compressed(os.path.join(HERE, "zebra.npz"), **arrays)
    dump("zebra_meta.json", meta)


CLI_CASES = [
    ["calls", "--kappa", "3", "--levels", "5"],
    ["calls", "--kappa", "inf", "--levels", "12"],
    ["predict", "--alpha", "0.00248", "--beta", "1.18e-6", "--kappa", "2", "--levels", "10"],
    ["predict", "--alpha", "0.00028", "--beta", "2e-8", "--kappa", "inf", "--levels", "12", "--nu", "2"],
    ["turning-point", "--alpha", "0.00248", "--beta", "1.18e-6", "--kappa", "inf"],
    ["turning-point", "--alpha", "0.0", "--beta", "1.18e-6", "--kappa", "2"],
    ["bench", "--kappa", "1,2,inf", "--levels", "4-6", "--reps", "0"],
    ["solve", "--levels", "7", "--kappa", "1", "--eps", "1e-4", "--phi", "45"],
    ["solve", "--levels", "6", "--kappa", "2", "--eps", "1e-4", "--phi", "45", "--solver", "pcg"],
    ["solve", "--levels", "5", "--kappa", "inf", "--eps", "0.1", "--phi", "30", "--out", "csv"],
    ["solve", "--levels", "5", "--kappa", "2", "--eps", "1e-4", "--phi", "45", "--max-cycles", "3"],
]
CLI_FIT_INPUT = "kappa,levels,ms\n1,4,0.1\n2,5,0.3\n3,6,0.9\ninf,7,2.5\n"


def gen_zebra9():
    """n = 9 zebra solves (the paper's Tables 5-8 solvers at a size the
    reference finishes in minutes): alternating zebra with full coarsening
    and zebra-x with y-semi-coarsening, kappa 2 / 3, eps 1e-5 and 1e-4,
    phi 45, error reduction 1e8 (cycle.py:303-366) -- pins the FMA build's
    partitioned line solver (kc_zebra.cuh k_zebra_solve_part) by counts and
    histories."""
    out = {}
    for sm, co in (("zebra-xy", "full"), ("zebra-x", "semi-y")):
        for eps in (1e-5, 1e-4):
            for kappa in (2, 3):
                problem, cfg = problem_config(9, kappa, eps=eps, smoother=_smoother(sm), coarsening=_coarsening(co))
                t0 = time.perf_counter()
                rep = kc.solve_standalone(problem, cfg, 1e8, max_cycles=3000)
                key = f"{sm}_{co}_n9_k{kappa}_eps{eps:g}"
                out[key] = {"smoother": sm, "coarsening": co, "n": 9, "kappa": kappa, "epsilon": eps, "phi": 45.0,
                            "status": rep.status, "iterations": rep.iterations,
                            "initial_error_norm": rep.initial_error_norm, "final_error_norm": rep.final_error_norm,
                            "per_cycle_reduction": rep.per_cycle_reduction,
                            "seconds": time.perf_counter() - t0}
                print(key, rep.status, rep.iterations, f"{time.perf_counter() - t0:.0f}s", flush=True)
                dump("zebra_n9.json", out)


def gen_cli():
    """The reference CLI (cli.py) on fixed argument lists: stdout and exit
    code; solve records without the run-dependent fields (wall_ms,
    timestamp, version)."""
    import contextlib
    import io
    from kcycle import cli
    out = []
    cases = [(c, None) for c in CLI_CASES] + [(["fit"], CLI_FIT_INPUT)]
    for argv, stdin in cases:
        buf = io.StringIO()
        old_in = sys.stdin
        if stdin is not None:
            sys.stdin = io.StringIO(stdin)
        try:
            with contextlib.redirect_stdout(buf):
                rc = cli.main(argv)
        finally:
            sys.stdin = old_in
        text = buf.getvalue()
        rec = {"argv": argv, "stdin": stdin, "exit": rc}
        if argv[0] == "solve" and "--out" not in argv:
            d = json.loads(text)
            d["result"].pop("wall_ms")
            rec["record"] = {"config": d["config"], "result": d["result"]}
        elif argv[0] == "solve":
            hdr, row = [line.split(",") for line in text.strip().splitlines()]
            rec["csv_header"] = hdr
            rec["csv_row"] = dict(zip(hdr, row))
            rec["csv_row"].pop("wall_ms")
        else:
            rec["stdout"] = text
        out.append(rec)
        print(argv, rc, flush=True)
    dump("cli.json", out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["small", "solve", "pcg", "costmodel", "cli", "zebra", "zebra9"])
    ap.add_argument("--n", type=int, default=12)
    ap.add_argument("--kappa", default="1")
    ap.add_argument("--cap", type=int, default=20000)
    a = ap.parse_args()
    print("reference kcycle", kcycle.__version__, "numpy", np.__version__, flush=True)
    if a.what == "costmodel":
        gen_costmodel()
        return
    if a.what == "cli":
        gen_cli()
        return
    if a.what == "zebra":
        gen_zebra()
        return
    if a.what == "zebra9":
        gen_zebra9()
        return
    if a.what == "small":
        gen_stencils()
        gen_kernels()
        gen_dry()
        gen_cycles()
        gen_solves_small()
        return
    kappa = INF if a.kappa in ("W", "inf") else int(a.kappa)
    if a.what == "solve":
        track_standalone(a.n, kappa, cap=a.cap, out_name=f"solve_n{a.n}_k{kname(kappa)}.json")
    else:
        track_pcg(a.n, kappa, cap=a.cap, out_name=f"pcg_n{a.n}_k{kname(kappa)}.json")


if __name__ == "__main__":
    main()
