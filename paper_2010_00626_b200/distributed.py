"""Multi-GPU kappa-cycles: row-strip decomposition + coarse agglomeration
(the reference is single-domain, cycle.py:18-19).

One process (rank) per GPU.  Every *distributed* level l (side >= world *
`min_rows`) is split into contiguous row strips; rank r owns fine rows
[a_r, b_r) with a_r even, so coarse row q (fine centre 2q+1, transfer.py:3-4)
belongs to the rank owning fine row 2q+1 and each finer level's strips are
exactly twice the coarser one's.  Halo rows (depth 2: a Jacobi sweep needs 1,
residual + full weighting of the last owned coarse row needs 2) are
exchanged with the neighbours before each stencil operation; the domain
boundary rows stay the zero Dirichlet ghosts.

Below the distributed levels the hierarchy is *agglomerated*: the restricted
right-hand side of the first coarse level is all-gathered, every rank runs
the remaining sub-cycle redundantly on the native single-GPU engine (graph +
persistent bottom kernel), and prolongs its own strip from its replica — no
scatter.  Stopping-test norms are per-rank partial sums + one allreduce.

Per-point arithmetic is the single-domain kernels' (bit-identical iterates);
only the norms are summed in a different order.

The driver is written against two small interfaces so the host logic can be
tested without GPUs (tests/test_distributed.py runs it with numpy strip ops,
in-process threads and torch.distributed/gloo):

* a communicator (`TorchComm` over torch.distributed -- NCCL on the B200
  box; `ThreadComm` for in-process ranks);
* a strip-ops backend (`CudaStripOps`: the C-ABI row-strip kernels of
  include/kcb200.h on torch CUDA tensors, plus `CudaCoarse` for the
  agglomerated levels on a CudaGridState).
"""

from __future__ import annotations

import math
import threading
import time
from dataclasses import dataclass

import numpy as np

from .costmodel import level_calls  # noqa: F401  (re-exported for planners)
from .cycle import CycleConfig, CycleStats, DryState, kappa_cycle
from .mesh import Coarsening, build_hierarchy
from .stencil import ProblemSpec, operator_hierarchy

HALO = 6  # halo rows per strip buffer: the fused passes need nu1 + 2 (pre) and nu2 (post)
KC_OX = 16
FUSE_MIN_M = 127  # narrower levels keep the per-op strip kernels (kc_engine.cu KC_FUSE_MIN_M)


def kc_pitch(m: int) -> int:
    """Row pitch (doubles) of a level with side m; mirrors kc_common.cuh."""
    return (KC_OX + m + 128 + 15) & ~15


# ---------------------------------------------------------------------------
# partition
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Plan:
    n: int
    world: int
    n_dist: int                       # levels 1..n_dist are distributed
    rows: tuple[tuple[tuple[int, int], ...], ...]  # rows[l-1][r] = (a, b) for distributed levels

    def side(self, level: int) -> int:
        return 2 ** (self.n - level + 1) - 1


def plan_partition(n: int, world: int, min_rows: int = 64) -> Plan:
    """Distributed levels: side >= world * min_rows (at least the finest level
    when n >= 2); strips even-aligned so coarse rows nest."""
    sides = [2 ** (n - l + 1) - 1 for l in range(1, n + 1)]
    n_dist = 0
    if world >= 1:  # world 1: one strip per level (the N > 1 code path on one device)
        for l in range(1, n):  # the coarsest level is never distributed
            if sides[l - 1] >= world * min_rows:
                n_dist = l
        if n_dist == 0 and n >= 2 and sides[0] >= 2 * world + 1:
            n_dist = 1
    rows = []
    if n_dist:
        mc = sides[n_dist - 1]
        cuts = [2 * ((r * (mc + 1)) // (2 * world)) for r in range(world)] + [mc]
        level_rows = [tuple((cuts[r], cuts[r + 1]) for r in range(world))]
        for l in range(n_dist - 1, 0, -1):  # finer levels: double, last rank takes the final row
            m = sides[l - 1]
            prev = level_rows[0]
            level_rows.insert(0, tuple((2 * a, 2 * b if r < world - 1 else m) for r, (a, b) in enumerate(prev)))
        rows = level_rows
    return Plan(n=n, world=world, n_dist=n_dist, rows=tuple(rows))


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------

class TorchComm:
    """torch.distributed: NCCL for CUDA tensors on the B200 box, gloo on CPU."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()

    def sendrecv(self, sends: dict, recvs: dict):
        """sends/recvs: {peer: tensor}; all posted at once (batch_isend_irecv)."""
        ops = []
        for peer, t in sends.items():
            ops.append(self.dist.P2POp(self.dist.isend, t.contiguous(), peer))
        for peer, t in recvs.items():
            ops.append(self.dist.P2POp(self.dist.irecv, t, peer))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()

    def allreduce_sum(self, t):
        self.dist.all_reduce(t)
        return t

    def allgather(self, t):
        """Equal-shape all_gather; returns a list of tensors."""
        import torch
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t.contiguous())
        return out


class ThreadComm:
    """In-process ranks (one thread each) exchanging tensors by reference-copy:
    used to run the decomposition on one device or on the CPU."""

    class _Shared:
        def __init__(self, world):
            self.world = world
            self.cv = threading.Condition()
            self.box = {}
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, shared: "ThreadComm._Shared", rank: int):
        self.s = shared
        self.rank = rank
        self.world = shared.world
        self.seq = 0

    @classmethod
    def group(cls, world: int):
        sh = cls._Shared(world)
        return [cls(sh, r) for r in range(world)]

    def sendrecv(self, sends: dict, recvs: dict):
        self.seq += 1
        with self.s.cv:
            for peer, t in sends.items():
                self.s.box[(self.rank, peer, self.seq)] = t.clone()
            self.s.cv.notify_all()
            for peer, t in recvs.items():
                key = (peer, self.rank, self.seq)
                while key not in self.s.box:
                    self.s.cv.wait()
                t.copy_(self.s.box.pop(key))

    def allreduce_sum(self, t):
        self.s.slots[self.rank] = t.clone()
        self.s.barrier.wait()
        total = self.s.slots[0].clone()
        for r in range(1, self.world):
            total += self.s.slots[r]
        self.s.barrier.wait()
        t.copy_(total)
        return t

    def allgather(self, t):
        self.s.slots[self.rank] = t.clone()
        self.s.barrier.wait()
        out = [self.s.slots[r].clone() for r in range(self.world)]
        self.s.barrier.wait()
        return out


# ---------------------------------------------------------------------------
# CUDA strip ops and agglomerated coarse solver
# ---------------------------------------------------------------------------

class CudaStripOps:
    """Row-strip kernels (kc_strip_*) on torch CUDA tensors of shape (rows, pitch)."""

    def __init__(self, device: int = 0):
        import torch

        from . import _native as N
        self.torch = torch
        self.N = N
        self.device = torch.device("cuda", device)

    def zeros(self, rows, pitch):
        return self.torch.zeros((rows, pitch), dtype=self.torch.float64, device=self.device)

    def _p(self, t, row):  # pointer to (row, column 0) of the interior
        return t.data_ptr() + 8 * (row * t.shape[1] + KC_OX)

    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def _w(self, w):
        self._wbuf = np.ascontiguousarray(np.asarray(w, dtype=np.float64).reshape(9))
        return self.N.dptr(self._wbuf)

    def jacobi(self, u, f, o, ny, nx, w, omega, zero):
        self.N.check(self.N.lib.kc_strip_jacobi(self._p(u, HALO), self._p(f, HALO), self._p(o, HALO), ny, nx,
                                                u.shape[1], self._w(w), omega, int(zero), self._stream()))

    def resid_restrict(self, u, f, fc, ncy, ncx, w, zero):
        self.N.check(self.N.lib.kc_strip_resid_restrict(self._p(u, HALO), self._p(f, HALO), self._p(fc, HALO),
                                                        ncy, ncx, u.shape[1], fc.shape[1], self._w(w), int(zero),
                                                        self._stream()))

    def prolong_add(self, v, vc, ny, nx, zero):
        self.N.check(self.N.lib.kc_strip_prolong_add(self._p(v, HALO), self._p(vc, HALO), ny, nx, v.shape[1],
                                                     vc.shape[1], int(zero), self._stream()))

    # fused passes (kc_strip_pre / kc_strip_post): the single-GPU streaming kernels on the strip
    def pre(self, u, f, uo, fc, ny, nx, crows, gy0, mg, w, omega, nu1, zero):
        self.N.check(self.N.lib.kc_strip_pre(self._p(u, HALO), self._p(f, HALO), self._p(uo, HALO), self._p(fc, HALO),
                                             ny, nx, u.shape[1], fc.shape[1], crows, gy0, mg, HALO, self._w(w),
                                             omega, nu1, int(zero), self._stream()))

    def post(self, u, f, uo, vc, ny, nx, crows, gy0, mg, w, omega, nu2, zero):
        self.N.check(self.N.lib.kc_strip_post(self._p(u, HALO), self._p(f, HALO), self._p(uo, HALO),
                                              self._p(vc, HALO), ny, nx, u.shape[1], vc.shape[1], crows, gy0, mg,
                                              HALO, HALO, self._w(w), omega, nu2, int(zero), self._stream()))

    def norms(self, v, f, ny, nx, w):
        out = self.torch.zeros(2, dtype=self.torch.float64, device=self.device)
        if ny > 0:
            self.N.check(self.N.lib.kc_strip_norms(self._p(v, HALO), self._p(f, HALO), ny, nx, v.shape[1],
                                                   self._w(w), out.data_ptr(), self._stream()))
        return out


class CudaCoarse:
    """The agglomerated levels as one native engine hierarchy (replicated per
    rank), issued on the caller's current stream without host waits (the
    engine follows torch's stream, so a distributed cycle can be captured
    into one CUDA graph)."""

    def __init__(self, problem: ProblemSpec, n_levels: int, ops, smoother, nu1, nu2, device=0):
        from .cycle import CudaGridState
        spec = build_hierarchy(n_levels, Coarsening.FULL_STANDARD)
        self.state = CudaGridState(spec, ops, smoother, nu1, nu2, device=device)
        self.m = spec.dims[0][0]

    def _bind_stream(self):
        import torch

        from . import _native as N
        N.check(N.lib.kc_set_stream(self.state._h, torch.cuda.current_stream().cuda_stream), self.state._h)

    def set_f(self, full):  # full: (m + 2*HALO, pitch) tensor with interior at (HALO, KC_OX)
        from . import _native as N
        self._bind_stream()
        ptr = full.data_ptr() + 8 * (HALO * full.shape[1] + KC_OX)
        N.check(N.lib.kc_set_device_async(self.state._h, 1, N.KC_WHICH_F, ptr, self.m, self.m, full.shape[1]),
                self.state._h)

    def zero_guess(self):
        self.state.zero_guess(1)

    def run(self, kappa):
        from . import _native as N
        N.check(N.lib.kc_cycle_enqueue(self.state._h, int(kappa)), self.state._h)

    def get_v(self, full):
        from . import _native as N
        ptr = full.data_ptr() + 8 * (HALO * full.shape[1] + KC_OX)
        N.check(N.lib.kc_get_device_async(self.state._h, 1, N.KC_WHICH_V, ptr, self.m, self.m, full.shape[1]),
                self.state._h)


# ---------------------------------------------------------------------------
# the SPMD solver
# ---------------------------------------------------------------------------

class _Strip:
    def __init__(self, ops, a, b, m, pitch):
        self.a, self.b, self.m = a, b, m
        self.ny = b - a
        rows = self.ny + 2 * HALO
        self.v = [ops.zeros(rows, pitch), ops.zeros(rows, pitch)]
        self.f = ops.zeros(rows, pitch)
        self.cur = 0
        self.vzero = True


class DistributedKappaSolver:
    """SPMD kappa-cycle over row strips (one instance per rank).

    `ops` / `make_coarse` select the device backend (CUDA by default);
    `comm` is a TorchComm (one process per GPU) or a ThreadComm.
    """

    def __init__(self, problem: ProblemSpec, config: CycleConfig, comm, ops=None, make_coarse=None,
                 min_rows: int = 64, device: int = 0, graphs: bool = True):
        if config.coarsening is not Coarsening.FULL_STANDARD:
            raise ValueError("distributed cycles support full coarsening only")
        self.problem, self.config, self.comm = problem, config, comm
        self.rank, self.world = comm.rank, comm.world
        self.n = config.n
        self.plan = plan_partition(self.n, self.world, min_rows)
        spec = build_hierarchy(self.n, config.coarsening)
        self.stencils = operator_hierarchy(problem, spec, config.coarse_op)
        self.w = [s.w for s in self.stencils]
        self.omega = config.smoother.omega
        self.nu1, self.nu2 = config.nu1, config.nu2
        self.ops = ops if ops is not None else CudaStripOps(device)
        self.strips = []
        for l in range(1, self.plan.n_dist + 1):
            a, b = self.plan.rows[l - 1][self.rank]
            m = self.plan.side(l)
            self.strips.append(_Strip(self.ops, a, b, m, kc_pitch(m)))
        nd = self.plan.n_dist
        self.nc = self.n - nd  # agglomerated levels
        mc = self.plan.side(nd + 1)
        if make_coarse is None:
            def make_coarse(levels, ws):
                return CudaCoarse(problem, levels, [self.stencils[nd + i] for i in range(levels)],
                                  config.smoother, self.nu1, self.nu2, device)
        self.coarse = make_coarse(self.nc, self.w[nd:])
        self.cfull = self.ops.zeros(mc + 2 * HALO, kc_pitch(mc))   # replicated level n_dist+1 (f, then v)
        self.vfull = self.ops.zeros(mc + 2 * HALO, kc_pitch(mc))
        self._stats_cache = {}
        # one CUDA graph per cycle counter (CUDA strips + NCCL + the native
        # coarse engine all on torch's stream); captured on the second call
        self._graphs_ok = (graphs and isinstance(self.ops, CudaStripOps) and isinstance(comm, TorchComm)
                           and isinstance(self.coarse, CudaCoarse))
        self._graphs = {}
        self._warm = set()
        if self._graphs_ok:
            import torch
            self._nrm = torch.zeros(2, dtype=torch.float64, device=self.ops.device)

    # -- data in/out -------------------------------------------------------
    def set_level1(self, which: str, full: np.ndarray):
        """Scatter a global finest-level array (every rank passes the same host array)."""
        s = self.strips[0]
        t = s.f if which == "f" else s.v[s.cur]
        rows = np.asarray(full, dtype=np.float64)[s.a:s.b]
        host = np.zeros((s.ny, t.shape[1]))
        host[:, KC_OX:KC_OX + s.m] = rows
        t[HALO:HALO + s.ny].copy_(self.ops.torch.from_numpy(host) if hasattr(self.ops, "torch") else host)
        if which == "v":
            s.vzero = False
        else:
            self._halo(s, s.f, HALO)

    def gather_level1(self) -> np.ndarray:
        """All-gather the finest v (every rank receives the full array)."""
        s = self.strips[0]
        self._materialize(s)
        t = s.v[s.cur]
        maxrows = max(b - a for a, b in self.plan.rows[0])
        buf = self.ops.zeros(maxrows, t.shape[1])
        buf[:s.ny].copy_(t[HALO:HALO + s.ny])
        parts = self.comm.allgather(buf)
        out = np.empty((s.m, s.m))
        for r, (a, b) in enumerate(self.plan.rows[0]):
            out[a:b] = parts[r][:b - a, KC_OX:KC_OX + s.m].cpu().numpy()
        return out

    # -- halo exchange -----------------------------------------------------
    def _halo(self, s: _Strip, t, depth: int):
        """Rows [0, depth) go up, [ny-depth, ny) go down; halos land in the ghost rows."""
        sends, recvs = {}, {}
        if self.world > 1:
            up, down = self.rank - 1, self.rank + 1
            if up >= 0:
                sends[up] = t[HALO:HALO + depth]
                recvs[up] = t[HALO - depth:HALO]
            if down < self.world:
                sends[down] = t[HALO + s.ny - depth:HALO + s.ny]
                recvs[down] = t[HALO + s.ny:HALO + s.ny + depth]
            # sent rows and ghost rows are disjoint row blocks (contiguous
            # views): receive straight into the ghost rows
            self.comm.sendrecv(sends, recvs)

    def _materialize(self, s: _Strip):
        if s.vzero:
            s.v[s.cur].zero_()
            s.vzero = False

    # -- one distributed routine call (Algorithm 3, cycle.py:204-220) -------
    def _relax(self, l: int, count: int):
        s = self.strips[l - 1]
        for _ in range(count):
            if not s.vzero:
                self._halo(s, s.v[s.cur], 1)
            self.ops.jacobi(s.v[s.cur], s.f, s.v[s.cur ^ 1], s.ny, s.m, self.w[l - 1], self.omega, s.vzero)
            s.vzero = False
            s.cur ^= 1

    def _fused(self, l: int) -> bool:
        """Fused strip passes at distributed level l: wide enough, nu within the
        buffers' halo, every rank's strip at least HALO rows deep."""
        return (hasattr(self.ops, "pre") and self.plan.side(l) >= FUSE_MIN_M and self.nu1 <= 4 and self.nu2 <= 4
                and self.nu1 + 2 <= HALO and self.nu2 + 1 <= HALO
                and min(b - a for a, b in self.plan.rows[l - 1]) >= HALO)

    def _cycle(self, l: int, kappa: int):
        s = self.strips[l - 1]
        nd = self.plan.n_dist
        fused = self._fused(l)
        if fused:  # nu1 sweeps + residual + full weighting in one pass (cycle.py:211-213)
            if not s.vzero:  # the last owned coarse row reaches nu1 + 2 fine rows below the strip
                self._halo(s, s.v[s.cur], self.nu1 + 2)
        else:
            self._relax(l, self.nu1)
            if not s.vzero:
                self._halo(s, s.v[s.cur], 2)
        if l < nd:  # restrict into the next distributed strip
            c = self.strips[l]
            if fused:
                self.ops.pre(s.v[s.cur], s.f, s.v[s.cur ^ 1], c.f, s.ny, s.m, c.ny, s.a, s.m, self.w[l - 1],
                             self.omega, self.nu1, s.vzero)
                if self.nu1 > 0:
                    s.cur ^= 1
                    s.vzero = False
            else:
                self.ops.resid_restrict(s.v[s.cur], s.f, c.f, c.ny, c.m, self.w[l - 1], s.vzero)
            self._halo(c, c.f, HALO)
            c.vzero = True
            self._cycle(l + 1, kappa)
            if kappa > 1:
                self._cycle(l + 1, kappa - 1)
            self._halo(c, c.v[c.cur], self.nu2 // 2 + 2)
            vc, vc_rows = c.v[c.cur], c.ny
        else:  # agglomerate: all-gather the coarse rows, replicated sub-cycle
            mc = self.plan.side(l + 1)
            q0, q1 = s.a // 2, (s.b // 2 if self.rank < self.world - 1 else mc)
            maxq = max((b // 2 if r < self.world - 1 else mc) - a // 2 for r, (a, b) in enumerate(self.plan.rows[l - 1]))
            part = self.ops.zeros(maxq + 2 * HALO, self.cfull.shape[1])
            if fused:
                self.ops.pre(s.v[s.cur], s.f, s.v[s.cur ^ 1], part, s.ny, s.m, q1 - q0, s.a, s.m, self.w[l - 1],
                             self.omega, self.nu1, s.vzero)
                if self.nu1 > 0:
                    s.cur ^= 1
                    s.vzero = False
            else:
                self.ops.resid_restrict(s.v[s.cur], s.f, part, q1 - q0, mc, self.w[l - 1], s.vzero)
            parts = self.comm.allgather(part)
            for r, (a, b) in enumerate(self.plan.rows[l - 1]):
                ra, rb = a // 2, (b // 2 if r < self.world - 1 else mc)
                self.cfull[HALO + ra:HALO + rb].copy_(parts[r][HALO:HALO + rb - ra])
            self.coarse.set_f(self.cfull)
            self.coarse.zero_guess()
            self.coarse.run(kappa)
            if kappa > 1:
                self.coarse.run(kappa - 1)
            self.coarse.get_v(self.vfull)
            vc = self.vfull[q0:]  # local coarse row 0 <-> global row q0 (ghost rows above)
            # view whose interior origin (row HALO) is coarse row q0: vfull row HALO + q0
            vc_rows = q1 - q0
        if fused:  # v + P vc and nu2 sweeps in one pass (cycle.py:219-220)
            if not s.vzero:
                self._halo(s, s.v[s.cur], max(self.nu2, 1))
            self.ops.post(s.v[s.cur], s.f, s.v[s.cur ^ 1], vc, s.ny, s.m, vc_rows, s.a, s.m, self.w[l - 1],
                          self.omega, self.nu2, s.vzero)
            s.cur ^= 1
            s.vzero = False
        else:
            self.ops.prolong_add(s.v[s.cur], vc, s.ny, s.m, s.vzero)
            s.vzero = False
            self._relax(l, self.nu2)

    def cycle(self, kappa: int | None = None, stats: CycleStats | None = None, with_norms: bool = False):
        """One kappa-cycle (run_cycle, cycle.py:261-263) over the decomposed hierarchy."""
        k = self.config.effective_kappa if kappa is None else min(kappa, self.n)
        if self.plan.n_dist == 0:
            raise ValueError("nothing to distribute: use the single-GPU engine (run_cycle)")
        self._run(k, with_norms and self._graphs_ok)
        if stats is not None:
            if k not in self._stats_cache:
                st = CycleStats.for_levels(self.n)
                kappa_cycle(DryState(self.n, self.nu1, self.nu2), 1, k, st)
                self._stats_cache[k] = st
            stats.absorb(self._stats_cache[k])

    def _host_state(self):
        return tuple((st.cur, st.vzero) for st in self.strips)

    def _body(self, k: int, with_norms: bool):
        self._cycle(1, k)
        if with_norms:  # ||v||^2, ||f - A v||^2 of the result into self._nrm (allreduced)
            s = self.strips[0]
            self._halo(s, s.v[s.cur], 1)
            t = self.ops.norms(s.v[s.cur], s.f, s.ny, s.m, self.w[0])
            self.comm.allreduce_sum(t)
            self._nrm.copy_(t)

    def _run(self, k: int, with_norms: bool = False):
        """One cycle (and optionally the norms of its result): eager on the
        first call per key, then captured once and replayed as a CUDA graph."""
        key = (k, with_norms)
        if self._graphs_ok and key in self._warm:
            g = self._graphs.get(key)
            if g is None:
                g = self._capture(key)
            if g is not None:
                g.replay()
                return
        self._body(k, with_norms)
        self._warm.add(key)

    def _capture(self, key):
        """Capture _body(*key) into a CUDA graph; None (eager from then on)
        when the cycle does not return the strips to their buffer parity (a
        replayed graph would read the wrong buffers) or cannot be captured."""
        import torch
        state0 = self._host_state()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(g):
                self._body(*key)
        except Exception:  # a backend that cannot be captured: stay eager
            ok = False
        else:
            ok = self._host_state() == state0
        if not ok:
            for st, (cur, vz) in zip(self.strips, state0):
                st.cur, st.vzero = cur, vz
            self._graphs_ok = False
            return None
        self._graphs[key] = g
        return g

    def norms(self) -> tuple[float, float]:
        """(||v||, ||f - A v||) of the finest level: partial sums + allreduce."""
        s = self.strips[0]
        self._materialize(s)
        self._halo(s, s.v[s.cur], 1)
        t = self.ops.norms(s.v[s.cur], s.f, s.ny, s.m, self.w[0])
        self.comm.allreduce_sum(t)
        e2, r2 = (float(x) for x in t.cpu().tolist())
        return math.sqrt(e2), math.sqrt(r2)

    def snapshot(self):
        """Device copy of the finest v strip (restore() puts it back): repeat a solve without host traffic."""
        s = self.strips[0]
        self._materialize(s)
        self._snap = s.v[s.cur].clone()

    def restore(self):
        s = self.strips[0]
        s.v[s.cur].copy_(self._snap)
        s.vzero = False

    def solve_standalone(self, target_reduction=1e8, max_cycles=10000, initial_guess=None, stop="error",
                         resident=False):
        """Distributed solve_standalone (cycle.py:303-366); every rank returns the same report.
        resident=True solves from the finest v/f already on the devices."""
        m = self.plan.side(1)
        if not resident:
            v0 = (np.random.default_rng(self.problem.seed).random((m, m)) if initial_guess is None
                  else np.asarray(initial_guess, dtype=np.float64))
            self.set_level1("v", v0)
            self.set_level1("f", np.zeros((m, m)))
        stats = CycleStats.for_levels(self.n)
        t0 = time.perf_counter()
        e, r = self.norms()
        err, res = [e], [r]
        meas = err if stop == "error" else res
        target = meas[0] / target_reduction
        status, it, streak = "max_cycles", 0, 0
        if meas[0] <= target:
            status = "converged"
        else:
            k = self.config.effective_kappa
            for it in range(1, max_cycles + 1):
                if self._graphs_ok:  # cycle + norms as one graph, one host read
                    self.cycle(k, stats=stats, with_norms=True)
                    e2, r2 = self._nrm.tolist()
                    e, r = math.sqrt(e2), math.sqrt(r2)
                else:
                    self.cycle(stats=stats)
                    e, r = self.norms()
                err.append(e)
                res.append(r)
                if meas[-1] <= target:
                    status = "converged"
                    break
                streak = streak + 1 if meas[-1] > meas[-2] else 0
                if streak >= 5:
                    status = "diverged"
                    break
        return {"status": status, "iterations": it, "err_hist": err, "res_hist": res, "stats": stats,
                "wall_ms": 1e3 * (time.perf_counter() - t0)}
