"""A short n=12 stand-alone solve (the device loop graph) for an ncu launch
list: the per-iteration kernels of the loop.  Usage: ncu_solve.py [kappa] [arith]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_00626_b200 as kc  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
arith = sys.argv[2] if len(sys.argv) > 2 else "fast"
st = kc.build_state(kc.ProblemSpec(1e-4, 45.0, seed=0), kc.CycleConfig(n=12, kappa=k), arith=arith)
st.v[0] = np.random.default_rng(0).random((4095, 4095))
st.snapshot()
st.launches_per_cycle(k)
for _ in range(2):
    st.restore()
    print(st.solve_device(k, "residual", 1e10, 4)[:3])
