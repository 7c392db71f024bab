"""Cycle time of the zebra / semi-coarsening solvers (paper solvers 3-6) at n.

  python tools/probe_zebra.py [n]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2010_00626_b200 import CycleConfig, ProblemSpec, build_state  # noqa: E402
from paper_2010_00626_b200.mesh import Coarsening  # noqa: E402
from paper_2010_00626_b200.smoother import SmootherKind, SmootherSpec  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
import os
arith = sys.argv[2] if len(sys.argv) > 2 else "exact"
p = ProblemSpec(1e-5, 45.0, seed=0)
for sm, co in ((SmootherKind.ZEBRA_ALTERNATING, Coarsening.FULL_STANDARD), (SmootherKind.ZEBRA_X, Coarsening.SEMI_Y),
               (SmootherKind.DAMPED_JACOBI, Coarsening.SEMI_Y)):
    for k in (1, 2):
        cfg = CycleConfig(n=n, kappa=k, smoother=SmootherSpec(sm, 0.8), coarsening=co)
        st = build_state(p, cfg, arith=arith)
        m = 2 ** n - 1
        st.v[0] = np.random.default_rng(0).random((m, m))
        st.run_cycles(k, 2)
        ms = st.time_cycles(k, 5) / 5
        print(f"{arith} {os.environ.get('KC_ZEBRA_TILED', '1')} {sm.value:9s} {co.value:6s} n={n} kappa={k}: {ms:.3f} ms/cycle, {st.launches_per_cycle(k)} kernels",
              flush=True)
        st.close()
