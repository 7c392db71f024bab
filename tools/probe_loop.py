"""Stand-alone loop overhead: ms per cycle of the bare cycle graph
(time_cycles) vs the device solve loop (solve_device, stop never firing),
n = 12, both builds, kappa = 2, 3."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_00626_b200 as kc  # noqa: E402

N = 60
for arith in (sys.argv[1:] or ["fast", "exact"]):
    st = kc.build_state(kc.ProblemSpec(1e-4, 45.0, seed=0), kc.CycleConfig(n=12, kappa=2), arith=arith)
    st.v[0] = np.random.default_rng(0).random((4095, 4095))
    st.snapshot()
    for k in (2, 3):
        st.run_cycles(k, 3)
        bare = st.time_cycles(k, N) / N
        st.restore()
        st.solve_device(k, "residual", 1e300, 5)
        best = 1e9
        for _ in range(3):
            st.restore()
            it, status, dms, _, _ = st.solve_device(k, "residual", 1e300, N)
            best = min(best, dms / it)
        print(f"{arith} kappa={k}: bare cycle {bare:.4f} ms, loop {best:.4f} ms/cycle, overhead {1e3 * (best - bare):.1f} us",
              flush=True)
    st.close()
