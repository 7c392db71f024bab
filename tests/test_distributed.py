"""Multi-rank kappa-cycles — host logic on the CPU.

The distributed driver (paper_2010_00626_b200.distributed) runs here with the
test-only numpy strip backend, first with in-process thread ranks, then as
world_size-2 torch.distributed/gloo processes.  Bar: iterates bit-identical
to the single-domain oracle (which is pinned to the reference), identical
iteration counts.  The same driver with the CUDA strip kernels is covered by
tests/test_gpu_parity.py (thread ranks on one B200).
"""

import math
import os
import threading

import numpy as np
import pytest
import torch

from dist_numpy_backend import NumpyCoarse, NumpyStripOps
from oracle import kcycle_oracle as O
from paper_2010_00626_b200 import CycleConfig, ProblemSpec
from paper_2010_00626_b200.distributed import DistributedKappaSolver, ThreadComm, plan_partition


def test_plan_partition_properties():
    for n in (5, 7, 9, 12, 14):
        for world in (1, 2, 3, 4, 8):
            plan = plan_partition(n, world, min_rows=16)
            if plan.n_dist == 0:
                continue
            for l in range(1, plan.n_dist + 1):
                m = plan.side(l)
                rows = plan.rows[l - 1]
                assert rows[0][0] == 0 and rows[-1][1] == m
                for r in range(world):
                    a, b = rows[r]
                    assert a % 2 == 0 and a <= b
                    if r + 1 < world:
                        assert rows[r + 1][0] == b
                if l > 1:  # nesting: fine strip = 2 x coarse strip
                    for (a, b), (ac, bc) in zip(plan.rows[l - 1], plan.rows[l - 2]):
                        assert ac == 2 * a
            assert plan.side(plan.n_dist) >= 2 * world + 1


def _run_threads(world, fn):
    comms = ThreadComm.group(world)
    out = [None] * world
    err = []

    def body(r):
        try:
            out[r] = fn(comms[r])
        except BaseException as exc:  # pragma: no cover - surfaced below
            err.append(exc)
            raise

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise err[0]
    return out


def _solver(comm, n, kappa, eps, phi, nu1=2, nu2=2, min_rows=8):
    problem = ProblemSpec(eps, phi, seed=0)
    cfg = CycleConfig(n=n, kappa=kappa, nu1=nu1, nu2=nu2)
    ws = O.hierarchy(eps, phi, n)

    def make_coarse(levels, wsub):
        return NumpyCoarse(ws[n - levels:], 0.8, nu1, nu2)

    return DistributedKappaSolver(problem, cfg, comm, ops=NumpyStripOps(), make_coarse=make_coarse,
                                  min_rows=min_rows)


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("kappa", [1, 2, 3])
def test_thread_ranks_bit_exact_vs_single_domain(world, kappa):
    n, eps, phi = 7, 1e-3, 30.0
    m = 2 ** n - 1
    rng = np.random.default_rng(world * 10 + kappa)
    v0, f0 = rng.random((m, m)), rng.standard_normal((m, m))
    h = O.Hierarchy(O.hierarchy(eps, phi, n))
    h.v[0], h.f[0] = v0.copy(), f0.copy()
    ref = []
    for _ in range(2):
        h.cycle(kappa)
        ref.append(h.v[0].copy())

    def fn(comm):
        s = _solver(comm, n, kappa, eps, phi)
        assert s.plan.n_dist >= 2  # several distributed levels + agglomeration
        s.set_level1("v", v0)
        s.set_level1("f", f0)
        got = []
        for _ in range(2):
            s.cycle()
            got.append(s.gather_level1())
        return got

    for got in _run_threads(world, fn):
        for c in range(2):
            assert np.array_equal(got[c], ref[c]), (world, kappa, c)


@pytest.mark.parametrize("nu1,nu2", [(1, 1), (2, 0), (0, 2), (3, 1)])
def test_thread_ranks_nu_variants(nu1, nu2):
    n, eps, phi, world, kappa = 6, 1e-4, 45.0, 2, 2
    m = 2 ** n - 1
    rng = np.random.default_rng(nu1 * 7 + nu2)
    v0, f0 = rng.random((m, m)), rng.random((m, m))
    h = O.Hierarchy(O.hierarchy(eps, phi, n), nu1=nu1, nu2=nu2)
    h.v[0], h.f[0] = v0.copy(), f0.copy()
    h.cycle(kappa)

    def fn(comm):
        s = _solver(comm, n, kappa, eps, phi, nu1, nu2, min_rows=4)
        s.set_level1("v", v0)
        s.set_level1("f", f0)
        s.cycle()
        return s.gather_level1()

    for got in _run_threads(world, fn):
        assert np.array_equal(got, h.v[0])


def test_thread_ranks_solve_counts():
    n, eps, phi, kappa = 6, 1e-4, 45.0, 2
    ref = O.standalone(eps, phi, n, kappa, target=1e8, stop="residual")

    def fn(comm):
        s = _solver(comm, n, kappa, eps, phi, min_rows=4)
        return s.solve_standalone(1e8, max_cycles=500, stop="residual")

    for rep in _run_threads(3, fn):
        assert rep["status"] == ref["status"]
        assert rep["iterations"] == ref["iterations"]
        rr = np.asarray(ref["res_hist"])
        assert np.max(np.abs(np.asarray(rep["res_hist"]) - rr) / rr) < 1e-12
        assert rep["stats"].visits == [O.level_calls(kappa, n)[l] * rep["iterations"] for l in range(n)]


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2010_00626_b200.distributed import TorchComm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, kappa = 6, 3
        m = 2 ** n - 1
        rng = np.random.default_rng(5)
        v0, f0 = rng.random((m, m)), rng.standard_normal((m, m))
        s = _solver(TorchComm(), n, kappa, 0.1, 45.0, min_rows=4)
        s.set_level1("v", v0)
        s.set_level1("f", f0)
        s.cycle()
        got = s.gather_level1()
        e, r = s.norms()
        q.put((rank, got, e, r))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_bit_exact():
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, kappa = 6, 3
    m = 2 ** n - 1
    rng = np.random.default_rng(5)
    v0, f0 = rng.random((m, m)), rng.standard_normal((m, m))
    h = O.Hierarchy(O.hierarchy(0.1, 45.0, n))
    h.v[0], h.f[0] = v0.copy(), f0.copy()
    h.cycle(kappa)
    e_ref = O.norm2(h.v[0])
    r_ref = O.norm2(O.residual(h.ws[0], h.v[0], h.f[0]))
    for rank, got, e, r in res:
        assert np.array_equal(got, h.v[0]), rank
        assert e == pytest.approx(e_ref, rel=1e-13) and r == pytest.approx(r_ref, rel=1e-13)


# ---------------------------------------------------------------------------
# distributed PCG and the device-side (batched) stop loops (kc_dist.cuh logic)
# ---------------------------------------------------------------------------

def _golden_pcg(n, kname):
    import json
    with open(os.path.join(os.path.dirname(__file__), "golden", "solves_small.json")) as fh:
        return json.load(fh)["pcg"][f"n{n}_k{kname}"]


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("kname,stop,tgt", [("1", "error", 1e8), ("2", "residual", 1e10), ("3", "error", 1e10),
                                            ("W", "residual", 1e10)])
def test_thread_ranks_pcg_counts_vs_reference(world, kname, stop, tgt):
    """Distributed pcg_solve (3 allreduced dots per iteration, alpha / beta /
    stop on the 'device' scalars) against the REAL reference's counts and
    histories (tests/golden/solves_small.json, made by make_golden.py)."""
    from conftest import check_pcg_hist
    n = 5
    g = _golden_pcg(n, kname)
    kappa = n if kname == "W" else int(kname)
    m = 2 ** n - 1
    x0 = np.random.default_rng(0).random((m, m))
    key = {("error", 1e8): "error_1e8", ("error", 1e10): "error_1e10", ("residual", 1e10): "residual_1e10"}[(stop, tgt)]

    def fn(comm):
        s = _solver(comm, n, kappa, 1e-4, 45.0, min_rows=4)
        return s.pcg_solve(np.zeros((m, m)), x0=x0, target_reduction=tgt, stop=stop, batch=3)

    for rep in _run_threads(world, fn):
        assert rep["status"] == "converged"
        assert rep["iterations"] == g["iters"][key]
        check_pcg_hist(rep["hist"], g["x_hist" if stop == "error" else "r_hist"])
        ref_rep = g["reference_reports"].get(key)
        if ref_rep is not None:
            assert rep["stats"].visits == ref_rep["visits"]


def test_thread_ranks_pcg_general_rhs_and_max_iterations():
    n, kappa, m = 5, 2, 31
    f = np.random.default_rng(12).random((m, m))
    ref = O.pcg(1e-4, 45.0, n, kappa, target=1e10, stop="residual", x0=np.zeros((m, m)), f=f)

    def fn(comm):
        s = _solver(comm, n, kappa, 1e-4, 45.0, min_rows=4)
        a = s.pcg_solve(f, target_reduction=1e10, stop="residual", batch=4)
        b = s.pcg_solve(f, target_reduction=1e10, stop="residual", max_iterations=3, batch=2)
        return a, b

    for a, b in _run_threads(2, fn):
        assert a["status"] == ref["status"] and a["iterations"] == ref["iterations"]
        assert np.allclose(a["solution"], ref["solution"], rtol=0, atol=1e-12 * np.max(np.abs(ref["solution"])))
        assert b["status"] == "max_cycles" and b["iterations"] == 3 and len(b["hist"]) == 4
        assert b["preconditioner_applications"] == 4  # the initial one + one per iteration


@pytest.mark.parametrize("batch", [1, 3, 8])
def test_thread_ranks_device_stop_loop_batches(batch):
    """The batched stand-alone loop: the stop fires inside a batch, the extra
    cycles are discarded, and the report (count, histories, solution) is the
    reference loop's, whatever the batch."""
    n, eps, phi, kappa = 6, 1e-4, 45.0, 3
    ref = O.standalone(eps, phi, n, kappa, target=1e8, stop="error")

    def fn(comm):
        s = _solver(comm, n, kappa, eps, phi, min_rows=4)
        rep = s.solve_standalone(1e8, max_cycles=500, stop="error", batch=batch)
        rep["solution"] = s.gather_level1()
        return rep

    for rep in _run_threads(2, fn):
        assert rep["status"] == ref["status"] == "converged"
        assert rep["iterations"] == ref["iterations"]
        ee = np.asarray(ref["err_hist"])
        assert len(rep["err_hist"]) == len(ee)
        assert np.max(np.abs(np.asarray(rep["err_hist"]) - ee) / ee) < 1e-12
        assert np.array_equal(rep["solution"], ref["solution"])


def test_thread_ranks_device_stop_max_cycles_and_divergence():
    n, kappa = 5, 2
    ref = O.standalone(1e-4, 45.0, n, kappa, target=1e10, max_cycles=7, stop="residual")

    def fn(comm):
        s = _solver(comm, n, kappa, 1e-4, 45.0, min_rows=4)
        return s.solve_standalone(1e10, max_cycles=7, stop="residual", batch=4)

    for rep in _run_threads(2, fn):
        assert rep["status"] == "max_cycles" and rep["iterations"] == 7 == ref["iterations"]
    # pure coarse-grid correction without smoothing never converges (test_cycle.py:225-233)
    ref = O.standalone(1.0, 0.0, 2, 1, target=1e8, max_cycles=40, seed=1, nu1=0, nu2=0)

    def fn2(comm):
        s = _solver(comm, 2, 1, 1.0, 0.0, nu1=0, nu2=0, min_rows=1)
        s.problem = ProblemSpec(1.0, 0.0, seed=1)
        return s.solve_standalone(1e8, max_cycles=40, batch=8)

    for rep in _run_threads(1, fn2):
        assert rep["status"] == ref["status"] and rep["iterations"] == ref["iterations"]


def _gloo_pcg_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2010_00626_b200.distributed import TorchComm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, kappa = 5, 2
        m = 2 ** n - 1
        x0 = np.random.default_rng(0).random((m, m))
        s = _solver(TorchComm(), n, kappa, 1e-4, 45.0, min_rows=4)
        rep = s.pcg_solve(np.zeros((m, m)), x0=x0, target_reduction=1e10, stop="residual", batch=4)
        sol = s.solve_standalone(1e8, max_cycles=500, stop="residual", batch=5)
        q.put((rank, rep["iterations"], rep["status"], rep["hist"], sol["iterations"], sol["status"]))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_pcg_and_device_stop():
    """world_size-2 torch.distributed/gloo processes: distributed PCG counts
    and histories equal the reference's; the batched stand-alone loop's
    count equals the oracle's."""
    import socket

    import torch.multiprocessing as mp

    from conftest import check_pcg_hist
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_pcg_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = _golden_pcg(5, "2")
    for rank, it, status, hist, sit, sst in res:
        assert status == "converged" and it == g["iters"]["residual_1e10"]
        check_pcg_hist(hist, g["r_hist"])
        assert sst == "converged"
    n5 = O.standalone(1e-4, 45.0, 5, 2, target=1e8, stop="residual")
    assert all(r[4] == n5["iterations"] for r in res), (res[0][4], n5["iterations"])


# ---------------------------------------------------------------------------
# interior / boundary windows of the overlapped fused strip passes
# ---------------------------------------------------------------------------

def _pre_deps(rows, crows, nu1, qlo, qhi):
    """Fine input rows the owned outputs of a pre window read (brute force)."""
    d = nu1 + 1
    need = set()
    for y in range(2 * qlo, min(2 * qhi, rows)):  # uo rows after nu1 sweeps
        if nu1:
            need.update(range(y - nu1, y + nu1 + 1))
    for q in range(qlo, min(qhi, crows)):  # residual rows 2q..2q+2, one more stencil, nu1 sweeps
        need.update(range(2 * q - d, 2 * q + 2 + d + 1))
    return need


def _post_deps(rows, nu2, qlo, qhi):
    need, cneed = set(), set()
    for y in range(2 * qlo, min(2 * qhi, rows)):
        for yy in range(y - nu2, y + nu2 + 1):
            need.add(yy)
            cneed.update({yy // 2 - 1, yy // 2} if yy % 2 == 0 else {yy // 2})
    return need, cneed


@pytest.mark.parametrize("rows,crows", [(86, 43), (84, 42), (85, 42), (512, 256), (17, 8), (30, 15)])
@pytest.mark.parametrize("nu", [0, 1, 2, 3, 4])
def test_overlap_windows_cover_and_stay_inside(rows, crows, nu):
    from paper_2010_00626_b200.distributed import post_windows, pre_windows
    win = pre_windows(rows, crows, nu)
    if win is not None:
        (qa, qb), outer = win
        assert outer == [(0, qa), (qb, crows + 1)] and 0 < qa < qb <= crows
        dep = _pre_deps(rows, crows, nu, qa, qb)
        assert min(dep) >= 0 and max(dep) <= rows - 1  # interior: no halo row
        assert min(_pre_deps(rows, crows, nu, qa - 1, qb)) < 0 or max(_pre_deps(rows, crows, nu, qa, qb + 1)) > rows - 1
    else:
        assert rows < 2 * (nu + 3)
    for vc_halo in (True, False):
        win = post_windows(rows, crows, nu, vc_halo)
        if win is None:
            continue
        (qa, qb), outer = win
        assert outer == [(0, qa), (qb, crows + 1)]
        dep, cdep = _post_deps(rows, nu, qa, qb)
        assert min(dep) >= 0 and max(dep) <= rows - 1
        if vc_halo:
            assert min(cdep) >= 0 and max(cdep) <= crows - 1
        # maximal: one more position on either side would read a halo row
        d0, c0 = _post_deps(rows, nu, qa - 1, qb) if qa > 0 else ({-1}, {-1})
        assert min(d0) < 0 or (vc_halo and min(c0) < 0)


def test_window_entry_points_reject_halo_reads_without_gpu():
    """kc_strip_*_window validate the window against hb / hbc before touching
    the device: one coarse row too far reads a halo row -> KC_EINVAL (the
    overlap split relies on hb = 0 meaning 'no halo row')."""
    import ctypes as C

    from paper_2010_00626_b200 import _native as N
    from paper_2010_00626_b200.distributed import post_windows, pre_windows
    w = (C.c_double * 9)(*([-1.0] * 4 + [8.0] + [-1.0] * 4))
    fake = 1 << 20  # never dereferenced: validation fails first
    rows, crows, nu = 86, 43, 2
    (qa, qb), _ = pre_windows(rows, crows, nu)
    for lo, hi in [(qa - 1, qb), (qa, qb + 1)]:
        rc = N.lib.kc_strip_pre_window(fake, fake, fake, fake, rows, 255, 288, 160, crows, 86, 255, 0, lo, hi, w, 0.8,
                                       nu, 0, None)
        assert rc == N.KC_EINVAL, (lo, hi)
    (qa, qb), _ = post_windows(rows, crows, nu, True)
    for lo, hi in [(qa - 1, qb), (qa, qb + 1)]:
        rc = N.lib.kc_strip_post_window(fake, fake, fake, fake, rows, 255, 288, 160, crows, 86, 255, 0, 0, lo, hi, w,
                                        0.8, nu, 0, None)
        assert rc == N.KC_EINVAL, (lo, hi)
