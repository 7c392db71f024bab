"""Per-(level, op) eager timings of one zebra cycle at n (default: zebra-x,
y-semi-coarsening, kappa 2, FMA build)."""
import collections
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_00626_b200 as kc  # noqa: E402
from paper_2010_00626_b200.mesh import Coarsening  # noqa: E402
from paper_2010_00626_b200.smoother import SmootherKind, SmootherSpec  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
sm = SmootherKind(sys.argv[2]) if len(sys.argv) > 2 else SmootherKind.ZEBRA_X
co = Coarsening(sys.argv[3]) if len(sys.argv) > 3 else Coarsening.SEMI_Y
k = int(sys.argv[4]) if len(sys.argv) > 4 else 2
arith = sys.argv[5] if len(sys.argv) > 5 else "fast"
cfg = kc.CycleConfig(n=n, kappa=k, smoother=SmootherSpec(sm, 0.8), coarsening=co)
st = kc.build_state(kc.ProblemSpec(1e-5, 45.0, seed=0), cfg, arith=arith)
nx, ny = st.spec.dims[0]
st.v[0] = np.random.default_rng(0).random((ny, nx))
acc = collections.defaultdict(float)
cnt = collections.Counter()
for p in st.profile_cycle(k):
    acc[(p["level"], p["op"])] += p["ms"]
    cnt[(p["level"], p["op"])] += 1
tot = sum(acc.values())
for key in sorted(acc):
    print(f"level {key[0]:2d} dims {st.spec.dims[key[0] - 1]} {key[1]:18s} x{cnt[key]:4d} {acc[key]:9.3f} ms")
print(f"total {tot:.2f} ms")
