"""A/B timing of the fused strip passes (kc_strip_pre / kc_strip_post) of two
engine libraries on one whole-level strip (4095^2, halo 6, nu = 2): the
multi-GPU path's kernels without any communication.
usage: ab_strip.py NAME=path.so [...]"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
m, mc, H, OX = 4095, 2047, 6, 16


def pitch(n):
    return ((n + OX + 127 + 15) // 16) * 16


P, Pc = pitch(m), pitch(mc)
dev = torch.device("cuda", 0)
u = torch.rand((m + 2 * H, P), dtype=torch.float64, device=dev)
f = torch.rand((m + 2 * H, P), dtype=torch.float64, device=dev)
uo = torch.zeros_like(u)
fc = torch.zeros((mc + 2 * H, Pc), dtype=torch.float64, device=dev)
for t in (u, f):
    t[:H].zero_(); t[H + m:].zero_(); t[:, :OX].zero_(); t[:, OX + m:].zero_()
w = (C.c_double * 9)(*([-0.1] * 4 + [1.0] + [-0.1] * 4))


def p(t, ps):
    return C.c_void_p(t.data_ptr() + 8 * (H * ps + OX))


res = {}
for spec in sys.argv[1:]:
    name, _, path = spec.partition("=")
    lib = C.CDLL(os.path.join(root, path))
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def pre():
        return lib.kc_strip_pre(p(u, P), p(f, P), p(uo, P), p(fc, Pc), m, m, P, Pc, mc, 0, m, H, w, C.c_double(0.8),
                                2, 0, st)

    def post():
        return lib.kc_strip_post(p(u, P), p(f, P), p(uo, P), p(fc, Pc), m, m, P, Pc, mc, 0, m, H, H, w,
                                 C.c_double(0.8), 2, 0, st)

    out = {}
    for nm, fn in (("pre", pre), ("post", post)):
        assert fn() == 0
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                fn()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) / 20 * 1e3)
        out[nm + "_us"] = round(best, 2)
    res[name] = out
    print(name, json.dumps(out), flush=True)
