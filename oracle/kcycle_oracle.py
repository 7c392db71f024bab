"""CPU oracle for the kappa-cycle hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package `kcycle`'s
algorithm for the hot path (arXiv 2010.00626; /root/reference/pkg/src/kcycle).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import it, and only as the checker or as the timed
CPU baseline -- never as the engine.  The product package
(paper_2010_00626_b200) never imports it and has no CPU fallback.

Parity pinning: every function here is checked against golden vectors that
tests/golden/make_golden.py produced by running the REAL reference in the
build container (tests/test_oracle.py): stencil hierarchies bit-exact,
per-kernel outputs bit-exact, whole-cycle iterates bit-exact (array data for
n=3/5, sha256 for n=7/9), solve histories and iteration counts.  The parity is
therefore pinned, not assumed.

Arithmetic contract, restated from the reference:
  * stencil application = scipy.ndimage.correlate(mode="constant", cval=0)
    (stencil.py:108-113): acc = 0, taps added in C order (dy outer, dx inner),
    each product and sum separately rounded, taps with |w| <= DBL_EPSILON
    skipped;
  * Jacobi u + (omega/center)*(f - Au)       smoother.py:95-100
  * full weighting / bilinear in numpy order  transfer.py:46-87
  * norm2 = np.linalg.norm (OpenBLAS ddot)    mesh.py:93-95
  * zebra line relaxation (smoother.py:107-135): even lines, then odd lines,
    each a tridiagonal solve of scipy.linalg.solve_banded((1,1)) = LAPACK
    dgtsv (Gaussian elimination with partial pivoting), restated in `gtsv`
    and pinned bit-exact against scipy itself (tests/test_oracle.py);
  * y-semi-coarsening transfers and the single-line coarsest solve
    (transfer.py:59-66, 84-86; cycle.py:191-200; smoother.py:71-92).
"""

from __future__ import annotations

import math
import sys

import numpy as np

DBL_EPS = sys.float_info.epsilon
INF = math.inf


# ---------------------------------------------------------------------------
# stencils (stencil.py:87-176)
# ---------------------------------------------------------------------------

def fine_stencil(epsilon: float, phi: float) -> np.ndarray:
    """stencil.py:87-105: rows south (dy=-1) to north (dy=+1)."""
    c = math.cos(math.radians(phi))
    s = math.sin(math.radians(phi))
    cross = 0.5 * (1.0 - epsilon) * c * s
    ns = -(epsilon * c * c + s * s)
    ew = -(c * c + epsilon * s * s)
    return np.array([[-cross, ns, cross], [ew, 2.0 * (1.0 + epsilon), ew], [cross, ns, -cross]])


def apply(w: np.ndarray, u: np.ndarray) -> np.ndarray:
    """stencil.py:108-113 via scipy.ndimage.correlate semantics (F2, F3)."""
    ny, nx = u.shape
    up = np.zeros((ny + 2, nx + 2))
    up[1:-1, 1:-1] = u
    acc = np.zeros((ny, nx))
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            wt = w[dy + 1, dx + 1]
            if abs(wt) <= DBL_EPS:
                continue
            acc = acc + wt * up[1 + dy:1 + dy + ny, 1 + dx:1 + dx + nx]
    return acc


def residual(w, u, f):
    """stencil.py:116-120."""
    return f - apply(w, u)


def prolong(c: np.ndarray) -> np.ndarray:
    """Bilinear prolongation, full coarsening (transfer.py:50-58)."""
    nyc, nxc = c.shape
    cp = np.zeros((nyc + 2, nxc + 2))
    cp[1:-1, 1:-1] = c
    out = np.zeros((2 * nyc + 1, 2 * nxc + 1))
    out[1::2, 1::2] = c
    out[1::2, 0::2] = 0.5 * (cp[1:-1, :-1] + cp[1:-1, 1:])
    out[0::2, 1::2] = 0.5 * (cp[:-1, 1:-1] + cp[1:, 1:-1])
    out[0::2, 0::2] = 0.25 * (cp[:-1, :-1] + cp[:-1, 1:] + cp[1:, :-1] + cp[1:, 1:])
    return out


def restrict(r: np.ndarray) -> np.ndarray:
    """Full weighting (transfer.py:75-83): (4C + 2(S+N+W+E) + (SW+SE+NW+NE)) / 16."""
    c = r[1::2, 1::2]
    s, n = r[0:-1:2, 1::2], r[2::2, 1::2]
    wv, e = r[1::2, 0:-1:2], r[1::2, 2::2]
    sw, se, nw, ne = r[0:-1:2, 0:-1:2], r[0:-1:2, 2::2], r[2::2, 0:-1:2], r[2::2, 2::2]
    return (4.0 * c + 2.0 * (s + n + wv + e) + (sw + se + nw + ne)) / 16.0


def prolong_semi(c: np.ndarray) -> np.ndarray:
    """Linear prolongation in y, y-semi-coarsening (transfer.py:59-66)."""
    nyc, nx = c.shape
    cp = np.zeros((nyc + 2, nx))
    cp[1:-1, :] = c
    out = np.zeros((2 * nyc + 1, nx))
    out[1::2, :] = c
    out[0::2, :] = 0.5 * (cp[:-1, :] + cp[1:, :])
    return out


def restrict_semi(r: np.ndarray) -> np.ndarray:
    """Full weighting in y (transfer.py:84-86): 0.25 (S + 2 C + N)."""
    return 0.25 * (r[0:-1:2, :] + 2.0 * r[1::2, :] + r[2::2, :])


FULL, SEMI_Y = "full", "semi-y"


def transfer(coarsening):
    return (prolong, restrict) if coarsening == FULL else (prolong_semi, restrict_semi)


def galerkin(w: np.ndarray, coarsening: str = FULL) -> np.ndarray:
    """R A P read off a 7x7 auxiliary coarse impulse (stencil.py:126-148)."""
    pro, res = transfer(coarsening)
    imp = np.zeros((7, 7))
    imp[3, 3] = 1.0
    resp = res(apply(w, pro(imp)))
    out = np.empty((3, 3))
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            out[dy + 1, dx + 1] = resp[3 - dy, 3 - dx]
    return out


def hierarchy(epsilon: float, phi: float, n: int, coarse_op: str = "galerkin", coarsening: str = FULL
              ) -> list[np.ndarray]:
    """stencil.py:151-176."""
    ws = [fine_stencil(epsilon, phi)]
    for l in range(1, n):
        ws.append(galerkin(ws[-1], coarsening) if coarse_op == "galerkin" else ws[0] * 0.25 ** l)
    return ws


def dims(n: int, coarsening: str = FULL) -> list[tuple[int, int]]:
    """(ny, nx) per level, finest first (mesh.py:56-73)."""
    if coarsening == FULL:
        return [(2 ** (n - l) - 1, 2 ** (n - l) - 1) for l in range(n)]
    return [(2 ** (n - l) - 1, 2 ** n - 1) for l in range(n)]


# ---------------------------------------------------------------------------
# smoother, coarsest solve (smoother.py:95-100, 138-148; cycle.py:182-190)
# ---------------------------------------------------------------------------

def jacobi(w, u, f, omega):
    center = float(w[1, 1])
    if center == 0.0:
        raise ValueError("zero center coefficient")
    return u + (omega / center) * (f - apply(w, u))


def gtsv(dl, d, du, b):
    """LAPACK dgtsv (scipy.linalg.solve_banded with l = u = 1): Gaussian
    elimination with partial pivoting, then back substitution; b is (n, k)."""
    dl, d, du, b = (np.array(a, dtype=float) for a in (dl, d, du, b))
    n = len(d)
    for i in range(n - 1):
        if abs(d[i]) >= abs(dl[i]):
            if d[i] == 0.0:
                raise np.linalg.LinAlgError("singular tridiagonal system")
            fact = dl[i] / d[i]
            d[i + 1] = d[i + 1] - fact * du[i]
            b[i + 1] = b[i + 1] - fact * b[i]
            if i < n - 2:
                dl[i] = 0.0
        else:  # interchange rows i and i+1
            fact = d[i] / dl[i]
            d[i] = dl[i]
            temp = d[i + 1]
            d[i + 1] = du[i] - fact * temp
            if i < n - 2:
                dl[i] = du[i + 1]
                du[i + 1] = -fact * dl[i]
            du[i] = temp
            temp = b[i].copy()
            b[i] = b[i + 1]
            b[i + 1] = temp - fact * b[i + 1]
    if d[n - 1] == 0.0:
        raise np.linalg.LinAlgError("singular tridiagonal system")
    b[n - 1] = b[n - 1] / d[n - 1]
    if n > 1:
        b[n - 2] = (b[n - 2] - du[n - 2] * b[n - 1]) / d[n - 2]
    for i in range(n - 3, -1, -1):
        b[i] = (b[i] - du[i] * b[i + 1] - dl[i] * b[i + 2]) / d[i]
    return b


def zebra(w, u, f, axis):
    """One zebra sweep with lines along `axis` (smoother.py:107-135): even
    lines then odd lines, rhs = f - (north/south part of A) u, each line a
    constant-coefficient tridiagonal solve.  y-lines run on the transposes."""
    if axis == "y":
        return zebra(np.ascontiguousarray(w.T), u.T, f.T, "x").T
    ny, nx = u.shape
    woff = w.copy()
    woff[1, :] = 0.0
    out = u.copy()
    for start in (0, 1):
        if start >= ny:
            break
        rhs = (f - apply(woff, out))[start::2]
        sol = gtsv(np.full(nx - 1, w[1, 0]), np.full(nx, w[1, 1]), np.full(nx - 1, w[1, 2]), rhs.T)
        out[start::2] = sol.T
    return out


JACOBI, ZEBRA_X, ZEBRA_Y, ZEBRA_XY = "jacobi", "zebra-x", "zebra-y", "zebra-xy"


def relax(w, u, f, omega, count, kind=JACOBI):
    """smoother.py:138-163."""
    if kind == JACOBI:
        for _ in range(count):
            u = jacobi(w, u, f, omega)
    elif kind in (ZEBRA_X, ZEBRA_Y):
        for _ in range(count):
            u = zebra(w, u, f, kind[-1])
    elif kind == ZEBRA_XY:
        if count % 2:
            raise ValueError("alternating zebra needs an even relaxation count")
        for _ in range(count // 2):
            u = zebra(w, u, f, "x")
            u = zebra(w, u, f, "y")
    else:
        raise ValueError(kind)
    return u


def thomas(lower, diag, upper, rhs):
    """smoother.py:71-92: forward elimination without pivoting."""
    m = len(diag)
    cp, dp = np.empty(m), np.empty(m)
    piv = diag[0]
    if piv == 0.0:
        raise np.linalg.LinAlgError("zero pivot in tridiagonal elimination")
    cp[0] = upper[0] / piv
    dp[0] = rhs[0] / piv
    for i in range(1, m):
        piv = diag[i] - lower[i] * cp[i - 1]
        if piv == 0.0:
            raise np.linalg.LinAlgError("zero pivot in tridiagonal elimination")
        cp[i] = upper[i] / piv
        dp[i] = (rhs[i] - lower[i] * dp[i - 1]) / piv
    x = np.empty(m)
    x[m - 1] = dp[m - 1]
    for i in range(m - 2, -1, -1):
        x[i] = dp[i] - cp[i] * x[i + 1]
    return x


def coarsest(w, f, coarsening=FULL):
    """cycle.py:182-200: 1x1 division, or one x-line Thomas solve (semi-y)."""
    ny, nx = f.shape
    if ny == 1 and nx == 1:
        center = float(w[1, 1])
        if center == 0.0:
            raise np.linalg.LinAlgError("singular coarsest operator")
        return f / center
    if coarsening == SEMI_Y and ny == 1:
        return thomas(np.full(nx, w[1, 0]), np.full(nx, w[1, 1]), np.full(nx, w[1, 2]), f[0].copy()).reshape(1, nx)
    raise ValueError(f"not a coarsest grid: {f.shape}")


def norm2(a) -> float:
    return float(np.linalg.norm(a))


def dot(a, b) -> float:
    return float(np.dot(a.ravel(), b.ravel()))


# ---------------------------------------------------------------------------
# kappa-cycle (Algorithm 3; cycle.py:204-220) on an explicit level list
# ---------------------------------------------------------------------------

class Hierarchy:
    """Per-level v, f and stencils; level index 0 = finest (cycle.py:144-179)."""

    def __init__(self, ws, omega=0.8, nu1=2, nu2=2, smoother=JACOBI, coarsening=FULL):
        self.ws = ws
        self.n = len(ws)
        self.omega, self.nu1, self.nu2 = omega, nu1, nu2
        self.smoother, self.coarsening = smoother, coarsening
        self.pro, self.res = transfer(coarsening)
        self.v = [np.zeros(d) for d in dims(self.n, coarsening)]
        self.f = [np.zeros(d) for d in dims(self.n, coarsening)]
        self.trace: list[tuple[int, int]] = []

    def _relax(self, l, count):
        self.v[l] = relax(self.ws[l], self.v[l], self.f[l], self.omega, count, self.smoother)

    def cycle(self, kappa: int, l: int = 0):
        self.trace.append((l + 1, kappa))
        if l == self.n - 1:
            self.v[l] = coarsest(self.ws[l], self.f[l], self.coarsening)
            return
        self._relax(l, self.nu1)
        self.f[l + 1] = self.res(residual(self.ws[l], self.v[l], self.f[l]))
        self.v[l + 1] = np.zeros_like(self.v[l + 1])
        self.cycle(kappa, l + 1)
        if kappa > 1:
            self.cycle(kappa - 1, l + 1)
        self.v[l] = self.v[l] + self.pro(self.v[l + 1])
        self._relax(l, self.nu2)


def eff_kappa(kappa, n):
    return n if kappa == INF else int(kappa)


def level_calls(kappa, n):
    """Per-level routine calls of one cycle (costmodel.py:138-153 closed form)."""
    k = eff_kappa(kappa, n)
    return [sum(math.comb(l - 1, j) for j in range(0, min(k - 1, l - 1) + 1)) for l in range(1, n + 1)]


def standalone(epsilon, phi, n, kappa, target=1e10, max_cycles=10000, seed=0, v0=None,
               stop="error", omega=0.8, nu1=2, nu2=2, track_residual=True, smoother=JACOBI, coarsening=FULL):
    """solve_standalone loop (cycle.py:320-353) with per-cycle error and true
    residual histories; `stop` picks the stopping measure."""
    h = Hierarchy(hierarchy(epsilon, phi, n, coarsening=coarsening), omega, nu1, nu2, smoother, coarsening)
    m = 2 ** n - 1
    h.v[0] = np.random.default_rng(seed).random((m, m)) if v0 is None else np.array(v0, dtype=float)
    k = eff_kappa(kappa, n)
    err = [norm2(h.v[0])]
    res = [norm2(residual(h.ws[0], h.v[0], h.f[0]))] if track_residual else []
    meas = err if stop == "error" else res
    tgt = meas[0] / target
    status, it, streak = "max_cycles", 0, 0
    if meas[0] <= tgt:
        status = "converged"
    else:
        for it in range(1, max_cycles + 1):
            h.cycle(k)
            err.append(norm2(h.v[0]))
            if track_residual:
                res.append(norm2(residual(h.ws[0], h.v[0], h.f[0])))
            if meas[-1] <= tgt:
                status = "converged"
                break
            streak = streak + 1 if meas[-1] > meas[-2] else 0
            if streak >= 5:
                status = "diverged"
                break
    return {"status": status, "iterations": it, "err_hist": err, "res_hist": res, "solution": h.v[0]}


def pcg(epsilon, phi, n, kappa, target=1e8, max_it=10000, seed=0, stop="error", x0=None, f=None):
    """pcg_solve loop (krylov.py:74-128) with one cycle per preconditioner application."""
    h = Hierarchy(hierarchy(epsilon, phi, n))
    m = 2 ** n - 1
    k = eff_kappa(kappa, n)
    w0 = h.ws[0]
    x = (np.random.default_rng(seed).random((m, m)) if x0 is None else np.array(x0, dtype=float))
    f = np.zeros((m, m)) if f is None else np.array(f, dtype=float)
    r = f - apply(w0, x)

    def prec(res):
        h.v[0] = np.zeros((m, m))
        h.f[0] = res.copy()
        h.cycle(k)
        return h.v[0].copy()

    def measure():
        return norm2(x) if stop == "error" else norm2(r)

    hist = [measure()]
    tgt = hist[0] / target
    status, it = "max_cycles", 0
    if hist[0] <= tgt:
        return {"status": "converged", "iterations": 0, "hist": hist, "solution": x}
    z = prec(r)
    rz = dot(r, z)
    if rz <= 0.0:
        return {"status": "breakdown", "iterations": 0, "hist": hist, "solution": x}
    p = z
    for it in range(1, max_it + 1):
        ap = apply(w0, p)
        pap = dot(p, ap)
        if pap <= 0.0:
            status = "breakdown"
            break
        alpha = rz / pap
        x = x + alpha * p
        r = r - alpha * ap
        hist.append(measure())
        if hist[-1] <= tgt:
            status = "converged"
            break
        z = prec(r)
        rz_next = dot(r, z)
        if rz_next <= 0.0:
            status = "breakdown"
            break
        p = z + (rz_next / rz) * p
        rz = rz_next
    return {"status": status, "iterations": it, "hist": hist, "solution": x}
