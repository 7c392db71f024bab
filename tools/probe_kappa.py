import time, numpy as np, sys
sys.path.insert(0, '.')
from paper_2010_00626_b200 import *
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
p = ProblemSpec(1e-4, 45.0, seed=0)
for k in (1, 2, 3, 4, n):
    cfg = CycleConfig(n=n, kappa=k)
    st = build_state(p, cfg)
    m = 2**n - 1
    st.v[0] = np.random.default_rng(0).random((m, m))
    t0 = time.time(); L = st.launches_per_cycle(k); tcap = time.time() - t0
    st.run_cycles(k, 3)
    ms = st.time_cycles(k, 20) / 20
    print(f"n={n} kappa={k}: {ms:.3f} ms/cycle, {L} kernels/cycle, capture {tcap*1e3:.0f} ms", flush=True)
    st.close()
