"""Device PCG time at n = 12 (both builds), kappa 2 and 3: ms per solve
(CUDA events inside kc_pcg), iterations.  usage: probe_pcg.py [fast|exact]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_00626_b200 as kc  # noqa: E402

arith = sys.argv[1] if len(sys.argv) > 1 else "fast"
n = 12
m = 2 ** n - 1
x0 = np.random.default_rng(0).random((m, m))
for k in (2, 3):
    cfg = kc.CycleConfig(n=n, kappa=k)
    st = kc.build_state(kc.ProblemSpec(1e-4, 45.0, seed=0), cfg, arith=arith)
    best = 1e9
    for _ in range(3):
        rep = kc.pcg_solve(st, np.zeros((m, m)), kc.PcgConfig(cycle=cfg, target_reduction=1e10, stop="residual"), x0=x0)
        best = min(best, rep.device_time_ms)
    print(f"{arith} kappa={k}: {rep.iterations} iterations, {best:.2f} ms, status {rep.status}", flush=True)
    st.close()
