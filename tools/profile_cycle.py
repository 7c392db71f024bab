"""Run a few n-level kappa-cycles of the engine for ncu (launch lists, full
captures of one kernel) and print the eager per-op profile.

  python tools/profile_cycle.py --n 12 --kappa 3 --cycles 1 [--eager]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2010_00626_b200 as kc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=12)
ap.add_argument("--kappa", default="3")
ap.add_argument("--cycles", type=int, default=1)
ap.add_argument("--eager", action="store_true", help="eager op-by-op cycles (kc_profile_cycle) instead of graphs")
ap.add_argument("--json", default="")
a = ap.parse_args()
n = a.n
k = n if a.kappa == "W" else int(a.kappa)
m = 2 ** n - 1
st = kc.build_state(kc.ProblemSpec(1e-4, 45.0, seed=0), kc.CycleConfig(n=n, kappa=k))
st.v[0] = np.random.default_rng(0).random((m, m))
prof = None
for _ in range(a.cycles):
    if a.eager:
        prof = st.profile_cycle(k)
    else:
        st.run_cycles(k, 1)
st.sync()
if prof is None:
    prof = st.profile_cycle(k)
tot = sum(p["ms"] for p in prof)
by = {}
for p in prof:
    key = (p["level"], p["op"])
    by.setdefault(key, [0, 0.0])
    by[key][0] += 1
    by[key][1] += p["ms"]
print(f"n={n} kappa={a.kappa}: eager cycle {tot:.3f} ms, {len(prof)} ops, graph kernels/cycle "
      f"{st.launches_per_cycle(k)}")
for (lev, op), (cnt, ms) in sorted(by.items()):
    print(f"  level {lev:2d} {op:18s} x{cnt:4d} {ms:8.3f} ms ({100 * ms / tot:5.1f}%)")
if a.json:
    with open(a.json, "w") as fh:
        json.dump({"n": n, "kappa": a.kappa, "ops": prof}, fh)
