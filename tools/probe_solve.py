"""Per-cycle cost of the device stand-alone loop vs bare cycle graphs (n=12).

  python tools/probe_solve.py [n] [kappa] [cycles]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2010_00626_b200 import CycleConfig, ProblemSpec, build_state  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cyc = int(sys.argv[3]) if len(sys.argv) > 3 else 50
st = build_state(ProblemSpec(1e-4, 45.0, seed=0), CycleConfig(n=n, kappa=k))
m = 2 ** n - 1
st.v[0] = np.random.default_rng(0).random((m, m))
st.snapshot()
st.run_cycles(k, 3)
print(f"bare cycle graph: {st.time_cycles(k, cyc) / cyc:.4f} ms/cycle", flush=True)
for rep in range(3):
    st.restore()
    it, status, dms, _, _ = st.solve_device(k, stop="residual", target_reduction=1e300, max_cycles=cyc)
    print(f"device solve loop: {it} cycles ({status}) {dms / it:.4f} ms/cycle", flush=True)
st.close()
