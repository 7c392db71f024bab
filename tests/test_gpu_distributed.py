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


@pytest.mark.parametrize("world,kname", [(2, "2"), (3, "3")])
def test_cuda_strips_device_stop_standalone_vs_reference(world, kname):
    n = 9
    g = load_json("solves_small.json")["standalone"][f"n{n}_k{kname}"]
    kappa = int(kname)

    def fn(comm):
        s = DistributedKappaSolver(ProblemSpec(1e-4, 45.0, seed=0), CycleConfig(n=n, kappa=kappa), comm, min_rows=16)
        return s.solve_standalone(1e10, max_cycles=2000, stop="residual", batch=6)

    for rep in _threads(world, fn):
        assert rep["status"] == "converged" and rep["iterations"] == g["iters_residual_1e10"]
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
        for _ in range(2):
            sol = s.solve_standalone(1e10, max_cycles=2000, stop="residual", batch=8)
            assert sol["status"] == "converged" and sol["iterations"] == gs["iters_residual_1e10"]
        assert s.graph_fallback is None, s.graph_fallback
        assert any(k[0] == "pcg" for k in s._graphs) and any(k[0] == "solve" for k in s._graphs)
    finally:
        dist.destroy_process_group()
