"""Three eager n=12 cycles for an ncu launch list (profile_cycle launches
every scheduled op once per cycle).  Usage: ncu_cycle.py [kappa] [exact|fast] [n]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_00626_b200 as kc  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
arith = sys.argv[2] if len(sys.argv) > 2 else "exact"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 12
m = 2 ** n - 1
st = kc.build_state(kc.ProblemSpec(1e-4, 45.0, seed=0), kc.CycleConfig(n=n, kappa=k), arith=arith)
st.v[0] = np.random.default_rng(0).random((m, m))
for _ in range(3):
    st.profile_cycle(k)
