"""Distributed solver on one GPU (world 1 over NCCL): per-cycle device/host
time and a cProfile of the host side.  Usage: probe_dist.py [n] [kappa]"""
import cProfile, os, pstats, sys, time
import numpy as np, torch, torch.distributed as dist
import paper_2010_00626_b200 as kc
from paper_2010_00626_b200.distributed import DistributedKappaSolver, TorchComm

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
kappa = int(sys.argv[2]) if len(sys.argv) > 2 else 2
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29534")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda:0"), rank=0, world_size=1)
m = 2 ** n - 1
s = DistributedKappaSolver(kc.ProblemSpec(1e-4, 45.0, seed=0), kc.CycleConfig(n=n, kappa=kappa), TorchComm(), min_rows=64)
s.set_level1("v", np.random.default_rng(0).random((m, m))); s.set_level1("f", np.zeros((m, m)))
for _ in range(3): s.cycle()
torch.cuda.synchronize()
N = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); e0.record()
for _ in range(N): s.cycle()
e1.record(); torch.cuda.synchronize()
print(f"n={n} kappa={kappa}: {e0.elapsed_time(e1) / N:.3f} ms/cycle device, {(time.perf_counter() - t0) * 1e3 / N:.3f} ms host")
pr = cProfile.Profile(); pr.enable()
for _ in range(N): s.cycle()
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
dist.destroy_process_group()
