"""Per-(level, op) eager timings of one kappa-cycle (CUDA events around each
scheduled op), several reps, min over reps.  Usage: probe_levels.py N KAPPA [exact|fast]"""
import os, sys, collections, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_00626_b200 as kc

n = int(sys.argv[1]); k = int(sys.argv[2])
arith = sys.argv[3] if len(sys.argv) > 3 else "exact"
st = kc.build_state(kc.ProblemSpec(1e-4, 45.0, seed=0), kc.CycleConfig(n=n, kappa=k), arith=arith)
m = 2 ** n - 1
st.v[0] = np.random.default_rng(0).random((m, m))
best = {}
for rep in range(5):
    acc = collections.defaultdict(list)
    for p in st.profile_cycle(k):
        acc[(p["level"], p["op"])].append(p["ms"])
    for key, v in acc.items():
        best[key] = min(best.get(key, (1e9, 0))[0], sum(v)), len(v)
tot = sum(v[0] for v in best.values())
for (lev, op), (ms, c) in sorted(best.items()):
    print(f"level {lev:2d} side {2**(n-lev+1)-1:5d} {op:12s} calls {c:3d} total {ms*1e3:8.1f} us  per call {ms*1e3/c:7.2f} us  {ms/tot:5.1%}")
print(f"total {tot*1e3:.1f} us")
