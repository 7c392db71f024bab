import sys, collections, numpy as np
import paper_2010_00626_b200 as kc
n = 12
for tile in (1, 0, 1, 0):
    st = kc.build_state(kc.ProblemSpec(1e-4, 45.0, seed=0), kc.CycleConfig(n=n, kappa=3))
    st.set_option("tile", tile)
    st.v[0] = np.random.default_rng(0).random((4095, 4095))
    best = {}
    for rep in range(5):
        acc = collections.defaultdict(list)
        for p in st.profile_cycle(3):
            acc[(p["level"], p["op"])].append(p["ms"])
        for key, v in acc.items():
            best[key] = min(best.get(key, 1e9), sum(v) / len(v))
    print("tile", tile, {k: round(v * 1e3, 2) for k, v in sorted(best.items()) if k[0] == 4 and k[1] != "zero_guess"})
