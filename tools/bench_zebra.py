"""The paper's zebra tables (Tables 5-8, RTX 3090) re-run on one B200:
14 levels (16383^2), eps = 1e-5, phi = 45 deg, error reduction 1e8, Galerkin
coarse operators, nu = (2, 2):

  Table 5  alternating zebra, full coarsening, stand-alone   (paper best: kappa 4, 199,501 ms, 463 cycles)
  Table 6  the same as the PCG preconditioner               (kappa 4, 26,439 ms, 53 iterations)
  Table 7  zebra-x, y-semi-coarsening, stand-alone           (kappa 3, 616,255 ms, 410 cycles)
  Table 8  the same as the PCG preconditioner               (kappa 2, 68,511 ms, 79 iterations)

Each row runs the paper's best kappa for that table in the FMA build (the
engine's headline build; its n = 9 counts equal the reference's,
tests/test_gpu_fast.py) and prints one JSON line.  Usage:
    python tools/bench_zebra.py [n] [arith]
"""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_00626_b200 as kc  # noqa: E402
from paper_2010_00626_b200.mesh import Coarsening  # noqa: E402
from paper_2010_00626_b200.smoother import SmootherKind, SmootherSpec  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 14
arith = sys.argv[2] if len(sys.argv) > 2 else "fast"
PAPER = {  # PAPER.md:745-827, phi = 45 column
    "table5": ("zebra-xy", "full", "standalone", 4, 199501, 463),
    "table6": ("zebra-xy", "full", "pcg", 4, 26439, 53),
    "table7": ("zebra-x", "semi-y", "standalone", 3, 616255, 410),
    "table8": ("zebra-x", "semi-y", "pcg", 2, 68511, 79),
}
problem = kc.ProblemSpec(1e-5, 45.0, seed=0)
out = {"n": n, "arith": arith, "epsilon": 1e-5, "phi": 45.0, "target": 1e8, "gpu": "B200", "rows": {}}
for name, (sm, co, mode, kappa, paper_ms, paper_it) in PAPER.items():
    cfg = kc.CycleConfig(n=n, kappa=kappa, smoother=SmootherSpec(SmootherKind(sm), 0.8), coarsening=Coarsening(co))
    st = kc.build_state(problem, cfg, arith=arith)
    m = 2 ** n - 1
    t0 = time.perf_counter()
    if mode == "standalone":
        rep = kc.solve_standalone(problem, cfg, 1e8, max_cycles=5000, state=st)
    else:
        x0 = np.random.default_rng(0).random((m, m))
        rep = kc.pcg_solve(st, np.zeros((m, m)), kc.PcgConfig(cycle=cfg, target_reduction=1e8, stop="error",
                                                              max_iterations=2000), x0=x0)
    wall = (time.perf_counter() - t0) * 1e3
    row = {"smoother": sm, "coarsening": co, "mode": mode, "kappa": kappa, "status": rep.status,
           "iterations": rep.iterations, "device_ms": rep.device_time_ms, "wall_ms": wall,
           "paper_rtx3090_ms": paper_ms, "paper_iterations": paper_it,
           "speedup_vs_paper": paper_ms / rep.device_time_ms if rep.device_time_ms else None}
    out["rows"][name] = row
    print(json.dumps({name: row}), flush=True)
    st.close()
print(json.dumps(out))
