"""TEST-ONLY numpy backend for the distributed driver (paper_2010_00626_b200.distributed).

Lets the multi-rank host logic (partition, halo exchange, agglomeration,
allreduce) run on the CPU with ThreadComm or torch.distributed/gloo.  The
strip arithmetic restates the oracle's (oracle/kcycle_oracle.py, itself
pinned to the reference) on strips with halo rows; the coarse replica is the
oracle Hierarchy.  Never imported by the package.
"""

import numpy as np
import torch

from oracle import kcycle_oracle as O
from paper_2010_00626_b200.distributed import HALO, KC_OX

EPS = np.finfo(float).eps


def _acc(w, up, ny, nx):
    """C-order 9-tap correlation of the padded view up (rows -1..ny, cols -1..nx)."""
    acc = np.zeros((ny, nx))
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            wt = w[dy + 1, dx + 1]
            if abs(wt) <= EPS:
                continue
            acc = acc + wt * up[1 + dy:1 + dy + ny, 1 + dx:1 + dx + nx]
    return acc


class NumpyStripOps:
    torch = torch

    def zeros(self, rows, pitch):
        return torch.zeros((rows, pitch), dtype=torch.float64)

    @staticmethod
    def _view(t, r0, r1, c0, c1):  # local rows [r0, r1), local cols [c0, c1)
        return t.numpy()[HALO + r0:HALO + r1, KC_OX + c0:KC_OX + c1]

    def jacobi(self, u, f, o, ny, nx, w, omega, zero):
        w = np.asarray(w).reshape(3, 3)
        fv = self._view(f, 0, ny, 0, nx)
        c = omega / float(w[1, 1])
        if zero:
            res = 0.0 + c * fv
        else:
            up = self._view(u, -1, ny + 1, -1, nx + 1)
            res = up[1:-1, 1:-1] + c * (fv - _acc(w, up, ny, nx))
        self._view(o, 0, ny, 0, nx)[...] = res

    def resid_restrict(self, u, f, fc, ncy, ncx, w, zero):
        w = np.asarray(w).reshape(3, 3)
        nyf, nxf = 2 * ncy + 1, 2 * ncx + 1
        fv = self._view(f, 0, nyf, 0, nxf)
        if zero:
            r = fv - 0.0 if False else fv.copy()
        else:
            up = self._view(u, -1, nyf + 1, -1, nxf + 1)
            r = fv - _acc(w, up, nyf, nxf)
        self._view(fc, 0, ncy, 0, ncx)[...] = O.restrict(r)

    def prolong_add(self, v, vc, ny, nx, zero):
        # coarse rows -1 .. ny//2 (+ ghost columns) around the strip
        mcy, mcx = ny // 2 + 1, (nx - 1) // 2
        cp = vc.numpy()[HALO - 1:HALO + mcy + 1, KC_OX - 1:KC_OX + mcx + 1]
        out = np.zeros((ny, nx))
        for y in range(ny):
            q = y >> 1
            for xs in (0, 1):
                xsl = slice(xs, nx, 2)
                p = np.arange(xs, nx, 2) >> 1
                if y & 1:
                    e = cp[q + 1, p + 1] if xs else 0.5 * (cp[q + 1, p] + cp[q + 1, p + 1])
                else:
                    if xs:
                        e = 0.5 * (cp[q, p + 1] + cp[q + 1, p + 1])
                    else:
                        e = 0.25 * (cp[q, p] + cp[q, p + 1] + cp[q + 1, p] + cp[q + 1, p + 1])
                out[y, xsl] = e
        view = self._view(v, 0, ny, 0, nx)
        view[...] = (0.0 if zero else view) + out

    def norms(self, v, f, ny, nx, w):
        w = np.asarray(w).reshape(3, 3)
        up = self._view(v, -1, ny + 1, -1, nx + 1)
        r = self._view(f, 0, ny, 0, nx) - _acc(w, up, ny, nx)
        vv = up[1:-1, 1:-1]
        return torch.tensor([float(np.sum(vv * vv)), float(np.sum(r * r))], dtype=torch.float64)


class NumpyCoarse:
    """Replicated coarse levels on the oracle Hierarchy."""

    def __init__(self, ws, omega, nu1, nu2):
        self.h = O.Hierarchy(ws, omega=omega, nu1=nu1, nu2=nu2)
        self.m = 2 ** len(ws) - 1

    def set_f(self, full):
        self.h.f[0] = full.numpy()[HALO:HALO + self.m, KC_OX:KC_OX + self.m].copy()

    def zero_guess(self):
        self.h.v[0] = np.zeros((self.m, self.m))

    def run(self, kappa):
        self.h.cycle(kappa)

    def get_v(self, full):
        full.numpy()[HALO:HALO + self.m, KC_OX:KC_OX + self.m] = self.h.v[0]


# ---------------------------------------------------------------------------
# device-side loop ops (kc_dist.cuh) restated in numpy, same slot layout
# ---------------------------------------------------------------------------
from paper_2010_00626_b200._native import DS, DS_PCG_MEAS, DS_PCG_PAP, DS_PCG_RZ, DS_PCG_RZ0, DS_SOLVE  # noqa: E402

_BREAKDOWN, _CONVERGED, _DIVERGED, _MAX = 3, 0, 1, 2


def _loop_ops(cls):
    def vector(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def _own(self, t, ny, nx):
        return self._view(t, 0, ny, 0, nx)

    def apply_dot(self, p, ap, ny, nx, w, part, scal, slot):
        if scal[DS["DONE"]] != 0:
            return
        w = np.asarray(w).reshape(3, 3)
        a = _acc(w, self._view(p, -1, ny + 1, -1, nx + 1), ny, nx)
        self._own(ap, ny, nx)[...] = a
        scal[slot] = float(np.sum(self._own(p, ny, nx) * a))

    def dot(self, a, b, ny, nx, part, scal, slot):
        if scal[DS["DONE"]] != 0:
            return
        scal[slot] = float(np.sum(self._own(a, ny, nx) * self._own(b, ny, nx)))

    def pcg_update_xr(self, x, r, p, ap, ny, nx, measure_x, part, scal):
        if scal[DS["DONE"]] != 0:
            return
        alpha = float(scal[DS["ALPHA"]])
        xv, rv = self._own(x, ny, nx), self._own(r, ny, nx)
        xv[...] = xv + alpha * self._own(p, ny, nx)
        rv[...] = rv - alpha * self._own(ap, ny, nx)
        v = xv if measure_x else rv
        scal[DS["MEAS"]] = float(np.sum(v * v))

    def pcg_update_p(self, p, z, ny, nx, scal):
        if scal[DS["DONE"]] != 0:
            return
        beta = float(scal[DS["BETA"]])
        pv = self._own(p, ny, nx)
        pv[...] = self._own(z, ny, nx) + beta * pv

    def residual(self, x, f, r, ny, nx, w):
        w = np.asarray(w).reshape(3, 3)
        self._own(r, ny, nx)[...] = self._own(f, ny, nx) - _acc(w, self._view(x, -1, ny + 1, -1, nx + 1), ny, nx)

    def copy_if(self, src, dst, ny, nx, scal):
        if scal[DS["JUST_DONE"]] != 0:
            self._own(dst, ny, nx)[...] = self._own(src, ny, nx)

    def dist_step(self, kind, scal, hist):
        """The reference's scalar decisions (the CUDA k_dist_step, restated)."""
        sc = scal.numpy()
        h = hist.numpy()
        was_done = sc[DS["DONE"]] != 0
        sc[DS["JUST_DONE"]] = 0.0
        if was_done:
            return

        def finish(status):
            sc[DS["STATUS"]], sc[DS["DONE"]], sc[DS["JUST_DONE"]] = status, 1.0, 1.0

        if kind == DS_PCG_RZ0:
            if not sc[DS["RZN"]] > 0.0:
                finish(_BREAKDOWN)
            else:
                sc[DS["RZ"]] = sc[DS["RZN"]]
        elif kind == DS_PCG_PAP:
            it = int(sc[DS["IT"]]) + 1
            sc[DS["IT"]] = it
            if not sc[DS["PAP"]] > 0.0:
                h[it] = np.nan
                finish(_BREAKDOWN)
            else:
                sc[DS["ALPHA"]] = sc[DS["RZ"]] / sc[DS["PAP"]]
        elif kind == DS_PCG_MEAS:
            it = int(sc[DS["IT"]])
            cur = float(np.sqrt(sc[DS["MEAS"]]))
            h[it] = cur
            if cur <= sc[DS["TARGET"]]:
                finish(_CONVERGED)
        elif kind == DS_PCG_RZ:
            rzn = sc[DS["RZN"]]
            if not rzn > 0.0:
                finish(_BREAKDOWN)
            elif int(sc[DS["IT"]]) >= int(sc[DS["MAXIT"]]):
                finish(_MAX)
            else:
                sc[DS["BETA"]] = rzn / sc[DS["RZ"]]
                sc[DS["RZ"]] = rzn
        elif kind == DS_SOLVE:
            it = int(sc[DS["IT"]])
            e, r = float(np.sqrt(sc[DS["E2"]])), float(np.sqrt(sc[DS["R2"]]))
            h[2 * it], h[2 * it + 1] = e, r
            cur = r if sc[DS["STOP_RESIDUAL"]] != 0 else e
            if it == 0:
                sc[DS["TARGET"]] = cur / sc[DS["REDUCTION"]]
            if cur <= sc[DS["TARGET"]]:
                finish(_CONVERGED)
            elif it > 0:
                streak = sc[DS["STREAK"]] + 1.0 if cur > sc[DS["PREV"]] else 0.0
                sc[DS["STREAK"]] = streak
                if streak >= 5.0:
                    finish(_DIVERGED)
            sc[DS["PREV"]] = cur
            if sc[DS["DONE"]] == 0:
                if it >= int(sc[DS["MAXIT"]]):
                    finish(_MAX)
                else:
                    sc[DS["IT"]] = it + 1

    for fn in (vector, _own, apply_dot, dot, pcg_update_xr, pcg_update_p, residual, copy_if, dist_step):
        setattr(cls, fn.__name__, fn)
    return cls


_loop_ops(NumpyStripOps)


def _norms_out(self, v, f, ny, nx, w, out=None):
    w = np.asarray(w).reshape(3, 3)
    up = self._view(v, -1, ny + 1, -1, nx + 1)
    r = self._view(f, 0, ny, 0, nx) - _acc(w, up, ny, nx)
    vv = up[1:-1, 1:-1]
    val = torch.tensor([float(np.sum(vv * vv)), float(np.sum(r * r))], dtype=torch.float64)
    if out is None:
        return val
    out.copy_(val)
    return out


NumpyStripOps.norms = _norms_out
