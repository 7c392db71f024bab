"""A/B timing of engine variants (tools/build_variant.sh): per variant, ms
per graph-launched cycle (n, kappa) and the eager per-(level, op) times of the
streaming levels.  usage: ab_stream.py N KAPPA ARITH NAME=path.so [...]
(NAME=default uses the in-tree library)"""
import json
import os
import subprocess
import sys

CHILD = r'''
import collections, ctypes, json, os, sys
import numpy as np
sys.path.insert(0, os.environ["KC_ROOT"])
if os.environ.get("AB_LENIENT") == "1":  # an older library: entry points it lacks become inert stubs
    _CDLL = ctypes.CDLL

    class _Lenient:
        def __init__(self, *a, **k):
            self._h = _CDLL(*a, **k)

        def __getattr__(self, name):
            try:
                return getattr(self._h, name)
            except AttributeError:
                f = lambda *a: 1  # noqa: E731
                f.restype = f.argtypes = None
                return f
    ctypes.CDLL = _Lenient
import paper_2010_00626_b200 as kc
n, k, arith = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
st = kc.build_state(kc.ProblemSpec(1e-4, 45.0, seed=0), kc.CycleConfig(n=n, kappa=k), arith=arith)
m = 2 ** n - 1
st.v[0] = np.random.default_rng(0).random((m, m))
st.run_cycles(k, 3)
cyc = min(st.time_cycles(k, 20) / 20 for _ in range(3))
best = {}
for rep in range(5):
    acc = collections.defaultdict(list)
    for p in st.profile_cycle(k):
        acc[(p["level"], p["op"])].append(p["ms"])
    for key, v in acc.items():
        best[key] = min(best.get(key, 1e9), sum(v) / len(v))
out = {"cycle_ms": cyc}
for (lev, op), ms in sorted(best.items()):
    if lev <= 3:
        out[f"L{lev}_{op}_us"] = round(ms * 1e3, 2)
print("JSON" + json.dumps(out))
'''

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n, k, arith = sys.argv[1], sys.argv[2], sys.argv[3]
res = {}
for spec in sys.argv[4:]:
    name, _, path = spec.partition("=")
    env = dict(os.environ, KC_ROOT=root)
    if path and path != "default":
        env["KCB200_LIB_FAST" if arith == "fast" else "KCB200_LIB"] = os.path.join(root, path)
    r = subprocess.run([sys.executable, "-c", CHILD, n, k, arith], env=env, capture_output=True, text=True)
    if r.returncode:
        res[name] = {"error": r.stderr[-800:]}
    else:
        res[name] = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("JSON")][-1][4:])
    print(name, json.dumps(res[name]), flush=True)
