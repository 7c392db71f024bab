"""Three eager n=12 cycles for an ncu launch list (profile_cycle launches
every scheduled op once per cycle).  Usage: ncu_cycle.py [kappa]"""
import sys

import numpy as np

import paper_2010_00626_b200 as kc

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
st = kc.build_state(kc.ProblemSpec(1e-4, 45.0, seed=0), kc.CycleConfig(n=12, kappa=k))
st.v[0] = np.random.default_rng(0).random((4095, 4095))
for _ in range(3):
    st.profile_cycle(k)
