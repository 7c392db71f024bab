"""A/B of the bottom-kernel launch shapes (env knobs read at kc_create):
ms per cycle for kappa = 1, 2, 3 at n = 12 in both arithmetic builds.
Usage: probe_bottom.py [arith] ; variants are listed below."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_00626_b200 as kc  # noqa: E402

arith = sys.argv[1] if len(sys.argv) > 1 else "fast"
n = 12
m = 2 ** n - 1
VARIANTS = {
    "entry127_cs16_min31": {},
    "no_deep127": {"KC_DEEP127": "0"},
    "no_frame_operators": {"KC_TINY_MV": "0"},
    "no_postpre": {"KC_POSTPRE": "0"},
    "postpre_stream": {"KC_POSTPRE_STREAM": "1"},
    "entry255_cs16_min31": {"KC_BOT_ENTRY": "255"},
    "entry127_cs16_min63": {"KC_BOT_MINSTRIP": "63"},
    "entry255_cs16_min63": {"KC_BOT_ENTRY": "255", "KC_BOT_MINSTRIP": "63"},
    "entry127_cs8_min31": {"KC_BOT_CS": "8"},
    "entry63_single": {"KC_BOT_CLUSTER": "0"},
}
KEYS = ("KC_DEEP127", "KC_BOT_ENTRY", "KC_BOT_MINSTRIP", "KC_BOT_CS", "KC_BOT_CLUSTER", "KC_TINY_MV", "KC_POSTPRE", "KC_POSTPRE_STREAM")
if len(sys.argv) > 2:
    VARIANTS = {k: VARIANTS[k] for k in sys.argv[2].split(",")}
v0 = np.random.default_rng(0).random((m, m))
only = [v for v in os.environ.get("PROBE_ONLY", "").split(",") if v]  # a subset of VARIANTS
for rep in range(2):
    for name, env in VARIANTS.items():
        if only and name not in only:
            continue
        for k in KEYS:
            os.environ.pop(k, None)
        os.environ.update(env)
        st = kc.build_state(kc.ProblemSpec(1e-4, 45.0, seed=0), kc.CycleConfig(n=n, kappa=2), arith=arith)
        st.v[0] = v0
        out = []
        for kap in (1, 2, 3, 4, n):
            st.run_cycles(kap, 3)
            out.append(st.time_cycles(kap, 40) / 40)
        print(f"{arith} {name:24s} " + " ".join(f"k{k}={t:.4f}" for k, t in zip((1, 2, 3, 4, "W"), out)), flush=True)
        st.close()
