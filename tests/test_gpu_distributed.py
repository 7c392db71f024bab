"""Distributed solvers with the CUDA strip kernels on one B200.

Thread ranks (ThreadComm, several ranks on one device) and an NCCL process
group of one rank (the N > 1 production path: torch.distributed, CUDA graph
capture of whole batches of iterations with NCCL allreduces inside) run the
distributed PCG (krylov.py:60-141; three allreduced dots per iteration,
alpha / beta / stop on the device) and the batched device-stop stand-alone
loop (cycle.py:303-366) against the REAL reference's goldens: identical
iteration counts, histories within the parity tolerances.
"""

import json
import os
import socket
import threading

import numpy as np
import pytest

from conftest import check_pcg_hist, load_json

pytestmark = pytest.mark.gpu

kc = pytest.importorskip("paper_2010_00626_b200")
from paper_2010_00626_b200 import CycleConfig, ProblemSpec  # noqa: E402
from paper_2010_00626_b200.distributed import DistributedKappaSolver, ThreadComm  # noqa: E402


def _threads(world, fn):
    comms = ThreadComm.group(world)
    out, err = [None] * world, []

    def body(r):
        try:
            out[r] = fn(comms[r])
        except BaseException as exc:
            err.append(exc)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not err, err
    return out


@pytest.mark.parametrize("world,n,kname,stop,tgt,key", [
    (2, 7, "2", "residual", 1e10, "residual_1e10"),
    (3, 7, "3", "error", 1e8, "error_1e8"),
    (2, 9, "1", "error", 1e10, "error_1e10"),
    (3, 9, "W", "residual", 1e10, "residual_1e10")])
def test_cuda_strips_pcg_vs_reference(world, n, kname, stop, tgt, key):
    g = load_json("solves_small.json")["pcg"][f"n{n}_k{kname}"]
    kappa = n if kname == "W" else int(kname)
    m = 2 ** n - 1
    x0 = np.random.default_rng(0).random((m, m))

    def fn(comm):
        s = DistributedKappaSolver(ProblemSpec(1e-4, 45.0, seed=0), CycleConfig(n=n, kappa=kappa), comm, min_rows=16)
        return s.pcg_solve(np.zeros((m, m)), x0=x0, target_reduction=tgt, stop=stop, batch=4)

    for rep in _threads(world, fn):
        assert rep["status"] == "converged" and rep["iterations"] == g["iters"][key]
        check_pcg_hist(rep["hist"], g["x_hist" if stop == "error" else "r_hist"])


@pytest.mark.parametrize("arith", ["exact", "fast"])
@pytest.mark.parametrize("world,kname", [(2, "2"), (3, "3")])
def test_cuda_strips_device_stop_standalone_vs_reference(world, kname, arith):
    """Both builds of the strip kernels and the agglomerated engine (the FMA
    build at the north star's bar: same counts, histories within 1e-10)."""
    n = 9
    g = load_json("solves_small.json")["standalone"][f"n{n}_k{kname}"]
    kappa = int(kname)

    def fn(comm):
        s = DistributedKappaSolver(ProblemSpec(1e-4, 45.0, seed=0), CycleConfig(n=n, kappa=kappa), comm, min_rows=16,
                                   arith=arith)
        assert s.ops.arith == arith and s.coarse.state.arith == arith
        return s.solve_standalone(1e10, max_cycles=2000, stop="residual", batch=6)

    for rep in _threads(world, fn):
        assert rep["status"] == "converged" and rep["iterations"] == g["iters_residual_1e10"]
        assert rep["gpu_launches"] > rep["iterations"]
        rr = np.asarray(g["res_hist"][: len(rep["res_hist"])])
        assert np.max(np.abs(np.asarray(rep["res_hist"]) - rr) / rr) < 1e-10


def test_nccl_world1_graph_batched_pcg_and_solve():
    """The production N > 1 path on one GPU: NCCL group of one rank, whole
    batches of PCG iterations / stand-alone cycles captured into CUDA graphs
    with the allreduces inside, one host read per batch."""
    import torch
    import torch.distributed as dist

    from paper_2010_00626_b200.distributed import TorchComm
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda:0"), rank=0, world_size=1)
    try:
        n, kappa = 9, 2
        m = 2 ** n - 1
        s = DistributedKappaSolver(ProblemSpec(1e-4, 45.0, seed=0), CycleConfig(n=n, kappa=kappa), TorchComm(),
                                   min_rows=32)
        gp = load_json("solves_small.json")["pcg"][f"n{n}_k2"]
        x0 = np.random.default_rng(0).random((m, m))
        for _ in range(2):  # the second call replays the captured batches
            rep = s.pcg_solve(np.zeros((m, m)), x0=x0, target_reduction=1e10, stop="residual", batch=4)
            assert rep["status"] == "converged" and rep["iterations"] == gp["iters"]["residual_1e10"]
            check_pcg_hist(rep["hist"], gp["r_hist"])
        gs = load_json("solves_small.json")["standalone"][f"n{n}_k2"]
        counts = []
        for _ in range(3):  # eager, captured, replayed: the same kernels each time
            sol = s.solve_standalone(1e10, max_cycles=2000, stop="residual", batch=8)
            assert sol["status"] == "converged" and sol["iterations"] == gs["iters_residual_1e10"]
            counts.append(sol["gpu_launches"])
        assert counts[0] == counts[1] == counts[2] and counts[0] > sol["iterations"], counts
        assert s.graph_fallback is None, s.graph_fallback
        assert any(k[0] == "pcg" for k in s._graphs) and any(k[0] == "solve" for k in s._graphs)
    finally:
        dist.destroy_process_group()


def _strip_bufs(ops, glob, a, rows, pitch, halo_fill=None):
    """A strip buffer holding global rows [a - HALO, a + rows + HALO) of glob
    (zero outside the domain); halo_fill replaces the halo rows (e.g. NaN)."""
    import torch

    from paper_2010_00626_b200.distributed import HALO, KC_OX
    mg, m = glob.shape
    host = np.zeros((rows + 2 * HALO, pitch))
    for r in range(rows + 2 * HALO):
        g = a - HALO + r
        if 0 <= g < mg:
            host[r, KC_OX:KC_OX + m] = glob[g]
    if halo_fill is not None:
        host[:HALO, KC_OX:KC_OX + m] = halo_fill
        host[HALO + rows:, KC_OX:KC_OX + m] = halo_fill
    return torch.from_numpy(host).to(ops.device)


@pytest.mark.parametrize("nu", [0, 1, 2, 3, 4])
def test_strip_windows_equal_whole_pass(nu):
    """kc_strip_pre_window / kc_strip_post_window: the interior window with
    hb = hbc = 0 reads no halo row (the halos are NaN during it) and, with the
    boundary windows after it, reproduces the whole-strip pass bit for bit --
    the overlap split of distributed.py."""
    from paper_2010_00626_b200.distributed import HALO, KC_OX, CudaStripOps, kc_pitch, post_windows, pre_windows
    from paper_2010_00626_b200.stencil import rotated_anisotropic_stencil
    ops = CudaStripOps(0)
    mg, mc = 255, 127
    P, Pc = kc_pitch(mg), kc_pitch(mc)
    rng = np.random.default_rng(nu)
    U, F, VC = rng.random((mg, mg)), rng.standard_normal((mg, mg)), rng.random((mc, mc))
    w = np.asarray(rotated_anisotropic_stencil(1e-4, 45.0).w, dtype=np.float64).reshape(9)
    for a, b in [(0, 86), (86, 170), (170, 255)]:
        rows = b - a
        crows = (b // 2 if b < mg else mc) - a // 2
        win = pre_windows(rows, crows, nu)
        assert win is not None
        outs = []
        for split in (False, True):
            u = _strip_bufs(ops, U, a, rows, P)
            f = _strip_bufs(ops, F, a, rows, P)
            uo, fc = ops.zeros(rows + 2 * HALO, P), ops.zeros(crows + 2 * HALO, Pc)
            args = (u, f, uo, fc, rows, mg, crows, a, mg, w, 0.8, nu, False)
            if not split:
                ops.pre(*args)
            else:
                un = _strip_bufs(ops, U, a, rows, P, halo_fill=np.nan)
                fn_ = _strip_bufs(ops, F, a, rows, P, halo_fill=np.nan)
                ops.pre(un, fn_, uo, fc, *args[4:], window=win[0], hb=0)
                for wd in win[1]:
                    ops.pre(*args, window=wd)
            outs.append((uo[HALO:HALO + rows, KC_OX:KC_OX + mg].cpu().numpy(),
                         fc[HALO:HALO + crows, KC_OX:KC_OX + mc].cpu().numpy()))
        assert np.isfinite(outs[1][1]).all()
        if nu:
            assert np.array_equal(outs[0][0], outs[1][0]), (a, b)
        assert np.array_equal(outs[0][1], outs[1][1]), (a, b)
        # post: v + P vc, nu sweeps; vc's halo exchanged (distributed coarse level) or local
        for vc_halo in (True, False):
            pw = post_windows(rows, crows, nu, vc_halo)
            assert pw is not None
            q0 = a // 2
            res = []
            for split in (False, True):
                u = _strip_bufs(ops, U, a, rows, P)
                f = _strip_bufs(ops, F, a, rows, P)
                vc = _strip_bufs(ops, VC, q0, crows, Pc)
                uo = ops.zeros(rows + 2 * HALO, P)
                args = (u, f, uo, vc, rows, mg, crows, a, mg, w, 0.8, nu, False)
                if not split:
                    ops.post(*args)
                else:
                    un = _strip_bufs(ops, U, a, rows, P, halo_fill=np.nan)
                    fn_ = _strip_bufs(ops, F, a, rows, P, halo_fill=np.nan)
                    vcn = _strip_bufs(ops, VC, q0, crows, Pc, halo_fill=np.nan) if vc_halo else vc
                    ops.post(un, fn_, uo, vcn, *args[4:], window=pw[0], hb=0, hbc=0 if vc_halo else HALO)
                    for wd in pw[1]:
                        ops.post(*args, window=wd)
                res.append(uo[HALO:HALO + rows, KC_OX:KC_OX + mg].cpu().numpy())
            assert np.isfinite(res[1]).all()
            assert np.array_equal(res[0], res[1]), (a, b, vc_halo)
