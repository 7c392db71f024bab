"""One device PCG solve at n = 12 (FMA build, kappa = 2) for an ncu capture of
the PCG vector kernels (the first A-block runs outside the conditional loop)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_00626_b200 as kc  # noqa: E402

n = 12
m = 2 ** n - 1
cfg = kc.CycleConfig(n=n, kappa=2)
st = kc.build_state(kc.ProblemSpec(1e-4, 45.0, seed=0), cfg, arith="fast")
x0 = np.random.default_rng(0).random((m, m))
if len(sys.argv) > 1 and sys.argv[1] == "host":
    # the host loop (a user preconditioner): every PCG vector kernel is an
    # ordinary launch ncu can time (z = r: Jacobi-free CG, a few iterations)
    rep = kc.pcg_solve(st, np.zeros((m, m)), kc.PcgConfig(cycle=cfg, target_reduction=1e10, stop="residual",
                                                          max_iterations=4), x0=x0, precondition=lambda r: r)
else:
    rep = kc.pcg_solve(st, np.zeros((m, m)), kc.PcgConfig(cycle=cfg, target_reduction=1e10, stop="residual"), x0=x0)
print(rep.status, rep.iterations)
