import numpy as np, paper_2010_00626_b200 as kc
st = kc.build_state(kc.ProblemSpec(1e-4, 45.0, seed=0), kc.CycleConfig(n=12, kappa=3))
st.v[0] = np.random.default_rng(0).random((4095, 4095))
for _ in range(3): st.profile_cycle(3)
