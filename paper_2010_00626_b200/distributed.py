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

from ._native import DS, DS_PART, DS_PCG_MEAS, DS_PCG_PAP, DS_PCG_RZ, DS_PCG_RZ0, DS_SLOTS, DS_SOLVE, STATUS_NAMES
from .costmodel import level_calls  # noqa: F401  (re-exported for planners)
from .cycle import CycleConfig, CycleStats, DryState, kappa_cycle
from .mesh import Coarsening, build_hierarchy
from .stencil import ProblemSpec, operator_hierarchy

HALO = 6  # halo rows per strip buffer: the fused passes need nu1 + 2 (pre) and nu2 (post)
KC_OX = 16
FUSE_MIN_M = 127  # narrower levels keep the per-op strip kernels (kc_engine.cu KC_FUSE_MIN_M)


def _floor2(a: int) -> int:
    return a // 2  # Python floors negative halves, as kc_engine.cu floor2


def pre_windows(rows: int, crows: int, nu1: int):
    """Interior / boundary coarse-row windows of a fused strip pre pass
    (kc_strip_pre_window): the interior window's outputs depend on the strip's
    own rows only (fine input rows [2 qa - D, 2 qb + D], D = nu1 + 1), so it
    runs with hb = 0 while the halo exchange is in flight; the boundary
    windows [0, qa) and [qb, crows + 1) run after it.  None: too few rows."""
    d = nu1 + 1
    qa, qb = (d + 1) // 2, min(crows, (rows - 1 - d) // 2)
    if qb - qa < 1:
        return None
    return (qa, qb), [(0, qa), (qb, crows + 1)]


def post_windows(rows: int, crows: int, nu2: int, vc_halo: bool):
    """The same for a fused strip post pass (kc_strip_post_window): fine rows
    [2q - nu2, 2q' - 1 + nu2] of u and, when vc's halo is exchanged too
    (vc_halo), the coarse rows those fine rows prolong from, inside the strip."""
    def lo_ok(q):
        lo = 2 * q - nu2
        clo = lo // 2 - 1 if lo % 2 == 0 else _floor2(lo)
        return lo >= 0 and (not vc_halo or clo >= 0)

    def hi_ok(q):
        hi = min(2 * q, rows) - 1 + nu2
        return hi <= rows - 1 and (not vc_halo or _floor2(hi) <= crows - 1)

    qa = 0
    while qa <= crows and not lo_ok(qa):
        qa += 1
    qb = crows + 1
    while qb > qa and not hi_ok(qb):
        qb -= 1
    if qb - qa < 1:
        return None
    return (qa, qb), [(0, qa), (qb, crows + 1)]


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

    @staticmethod
    def _settle(ts):
        """CUDA tensors: wait for this thread's current stream, so a copy made
        on one rank's stream is complete before another rank's stream (the
        overlap side stream, say) reads it or the allocator reuses it."""
        for t in ts:
            if getattr(t, "is_cuda", False):
                import torch
                torch.cuda.current_stream(t.device).synchronize()
                return

    def sendrecv(self, sends: dict, recvs: dict):
        self.seq += 1
        with self.s.cv:
            boxed = {peer: t.clone() for peer, t in sends.items()}
            self._settle(boxed.values())
            for peer, t in boxed.items():
                self.s.box[(self.rank, peer, self.seq)] = t
            self.s.cv.notify_all()
            for peer, t in recvs.items():
                key = (peer, self.rank, self.seq)
                while key not in self.s.box:
                    self.s.cv.wait()
                src = self.s.box.pop(key)
                t.copy_(src)
                self._settle([t])

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
    """Row-strip kernels (kc_strip_*) on torch CUDA tensors of shape (rows, pitch),
    from the exact (bit-identical to the reference) or the fast (FMA) build."""

    def __init__(self, device: int = 0, arith: str | None = None):
        import torch

        from . import _native as N
        self.torch = torch
        self.N = N
        self.arith = N.default_arith() if arith is None else arith
        self.lib = N.lib_for(self.arith)
        self.device = torch.device("cuda", device)
        self.launches = 0

    def _chk(self, rc, kernels: int = 1):
        self.N.check(rc, None, self.lib)  # the error text lives in the library that failed
        self.launches += kernels  # kernels the call enqueued (bench gpu_launches)

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
        self._chk(self.lib.kc_strip_jacobi(self._p(u, HALO), self._p(f, HALO), self._p(o, HALO), ny, nx,
                                                u.shape[1], self._w(w), omega, int(zero), self._stream()))

    def resid_restrict(self, u, f, fc, ncy, ncx, w, zero):
        self._chk(self.lib.kc_strip_resid_restrict(self._p(u, HALO), self._p(f, HALO), self._p(fc, HALO),
                                                        ncy, ncx, u.shape[1], fc.shape[1], self._w(w), int(zero),
                                                        self._stream()))

    def prolong_add(self, v, vc, ny, nx, zero):
        self._chk(self.lib.kc_strip_prolong_add(self._p(v, HALO), self._p(vc, HALO), ny, nx, v.shape[1],
                                                     vc.shape[1], int(zero), self._stream()))

    # fused passes (kc_strip_pre / kc_strip_post): the single-GPU streaming kernels on the strip;
    # window = (q_lo, q_hi): only those coarse-row chunk positions (kc_strip_*_window), reading
    # no more than hb fine / hbc coarse halo rows
    def pre(self, u, f, uo, fc, ny, nx, crows, gy0, mg, w, omega, nu1, zero, window=None, hb=HALO):
        args = (self._p(u, HALO), self._p(f, HALO), self._p(uo, HALO), self._p(fc, HALO), ny, nx, u.shape[1],
                fc.shape[1], crows, gy0, mg)
        if window is None:
            self._chk(self.lib.kc_strip_pre(*args, HALO, self._w(w), omega, nu1, int(zero), self._stream()))
        else:
            self._chk(self.lib.kc_strip_pre_window(*args, hb, window[0], window[1], self._w(w), omega, nu1,
                                                   int(zero), self._stream()))

    def post(self, u, f, uo, vc, ny, nx, crows, gy0, mg, w, omega, nu2, zero, window=None, hb=HALO, hbc=HALO):
        args = (self._p(u, HALO), self._p(f, HALO), self._p(uo, HALO), self._p(vc, HALO), ny, nx, u.shape[1],
                vc.shape[1], crows, gy0, mg)
        if window is None:
            self._chk(self.lib.kc_strip_post(*args, HALO, HALO, self._w(w), omega, nu2, int(zero), self._stream()))
        else:
            self._chk(self.lib.kc_strip_post_window(*args, hb, hbc, window[0], window[1], self._w(w), omega, nu2,
                                                    int(zero), self._stream()))

    def norms(self, v, f, ny, nx, w, out=None):
        """(sum v^2, sum (f - A v)^2) over the strip into `out` (2 doubles; new tensor if None)."""
        if out is None:
            out = self.torch.zeros(2, dtype=self.torch.float64, device=self.device)
        if ny > 0:
            self._chk(self.lib.kc_strip_norms(self._p(v, HALO), self._p(f, HALO), ny, nx, v.shape[1],
                                                   self._w(w), out.data_ptr(), self._stream()), 2)
        else:
            out.zero_()
        return out

    # -- device-side loops (kc_dist.cuh): scalars in `scal`, KC_DS_* slots --
    def vector(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device=self.device)

    def apply_dot(self, p, ap, ny, nx, w, part, scal, slot):
        self._chk(self.lib.kc_strip_apply_dot(self._p(p, HALO), self._p(ap, HALO), ny, nx, p.shape[1], self._w(w),
                                                   part.data_ptr(), scal.data_ptr(), slot, self._stream()), 2)

    def dot(self, a, b, ny, nx, part, scal, slot):
        self._chk(self.lib.kc_strip_dot(self._p(a, HALO), self._p(b, HALO), ny, nx, a.shape[1], part.data_ptr(),
                                             scal.data_ptr(), slot, self._stream()), 2)

    def pcg_update_xr(self, x, r, p, ap, ny, nx, measure_x, part, scal):
        self._chk(self.lib.kc_strip_pcg_update_xr(self._p(x, HALO), self._p(r, HALO), self._p(p, HALO),
                                                       self._p(ap, HALO), ny, nx, x.shape[1], int(measure_x),
                                                       part.data_ptr(), scal.data_ptr(), self._stream()), 2)

    def pcg_update_p(self, p, z, ny, nx, scal):
        self._chk(self.lib.kc_strip_pcg_update_p(self._p(p, HALO), self._p(z, HALO), ny, nx, p.shape[1],
                                                      scal.data_ptr(), self._stream()))

    def residual(self, x, f, r, ny, nx, w):
        self._chk(self.lib.kc_strip_residual(self._p(x, HALO), self._p(f, HALO), self._p(r, HALO), ny, nx,
                                                  x.shape[1], self._w(w), self._stream()))

    def copy_if(self, src, dst, ny, nx, scal):
        self._chk(self.lib.kc_strip_copy_if(self._p(src, HALO), self._p(dst, HALO), ny, nx, src.shape[1],
                                                 scal.data_ptr(), self._stream()))

    def dist_step(self, kind, scal, hist):
        self._chk(self.lib.kc_dist_step(kind, scal.data_ptr(), hist.data_ptr(), self._stream()))


class CudaCoarse:
    """The agglomerated levels as one native engine hierarchy (replicated per
    rank), issued on the caller's current stream without host waits (the
    engine follows torch's stream, so a distributed cycle can be captured
    into one CUDA graph)."""

    def __init__(self, problem: ProblemSpec, n_levels: int, ops, smoother, nu1, nu2, device=0, arith=None):
        from .cycle import CudaGridState
        spec = build_hierarchy(n_levels, Coarsening.FULL_STANDARD)
        self.state = CudaGridState(spec, ops, smoother, nu1, nu2, device=device, arith=arith)
        self.lib = self.state._lib
        self.launches = 0
        # kernels of one cycle per counter, counted now while the handle still
        # has its own stream (kc_cycle_launches captures a graph on it)
        self.levels = n_levels
        self._per_cycle = {k: self.state.launches_per_cycle(k) for k in range(1, n_levels + 1)}
        self.m = spec.dims[0][0]

    def _bind_stream(self):
        import torch

        from . import _native as N
        N.check(self.lib.kc_set_stream(self.state._h, torch.cuda.current_stream().cuda_stream), self.state._h,
                self.lib)

    def set_f(self, full):  # full: (m + 2*HALO, pitch) tensor with interior at (HALO, KC_OX)
        from . import _native as N
        self._bind_stream()
        ptr = full.data_ptr() + 8 * (HALO * full.shape[1] + KC_OX)
        N.check(self.lib.kc_set_device_async(self.state._h, 1, N.KC_WHICH_F, ptr, self.m, self.m, full.shape[1]),
                self.state._h, self.lib)

    def zero_guess(self):
        self.state.zero_guess(1)

    def run(self, kappa):
        from . import _native as N
        N.check(self.lib.kc_cycle_enqueue(self.state._h, int(kappa)), self.state._h, self.lib)
        self.launches += self._per_cycle[max(1, min(int(kappa), self.levels))]

    def get_v(self, full):
        from . import _native as N
        ptr = full.data_ptr() + 8 * (HALO * full.shape[1] + KC_OX)
        N.check(self.lib.kc_get_device_async(self.state._h, 1, N.KC_WHICH_V, ptr, self.m, self.m, full.shape[1]),
                self.state._h, self.lib)


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
        self.fpend = False  # f's halo rows still to exchange (restricted into, not yet exchanged)


class DistributedKappaSolver:
    """SPMD kappa-cycle over row strips (one instance per rank).

    `ops` / `make_coarse` select the device backend (CUDA by default);
    `comm` is a TorchComm (one process per GPU) or a ThreadComm.
    """

    def __init__(self, problem: ProblemSpec, config: CycleConfig, comm, ops=None, make_coarse=None,
                 min_rows: int = 64, device: int = 0, graphs: bool = True, overlap: bool | None = None,
                 arith: str | None = None):
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
        self.ops = ops if ops is not None else CudaStripOps(device, arith)
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
                                  config.smoother, self.nu1, self.nu2, device, getattr(self.ops, "arith", arith))
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
        self._key_launches = {}  # kernels one call of a graphed body enqueues
        self._replayed = 0       # kernels launched by graph replays
        self.graph_fallback = None
        if self._graphs_ok:
            import torch
            self._nrm = torch.zeros(2, dtype=torch.float64, device=self.ops.device)
        # halo exchange overlapped with the interior rows of the fused strip
        # passes (a side stream; default: on with CUDA strips and > 1 rank;
        # True forces the interior / boundary split even without exchanges)
        cuda = isinstance(self.ops, CudaStripOps)
        self.overlap = (cuda and self.world > 1) if overlap is None else (bool(overlap) and cuda)
        self._side = None
        if self.overlap:
            import torch
            self._side = torch.cuda.Stream(device=self.ops.device, priority=-1)

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

    def _exchange_then(self, exchanges, whole, inner, outer):
        """Run the halo exchanges, then a fused strip pass.  With overlap the
        exchanges go to a side stream (forked from and joined back into the
        current stream, so a captured graph keeps the order) while the pass's
        interior window `inner()` runs on the current stream; the boundary
        windows `outer()` follow the join.  Otherwise exchange, then `whole()`."""
        if not self.overlap or inner is None:
            for ex in exchanges:
                self._halo(*ex)
            whole()
            return
        torch = self.ops.torch
        main = torch.cuda.current_stream(self.ops.device)
        side = self._side
        if exchanges:
            side.wait_stream(main)
            with torch.cuda.stream(side):
                for ex in exchanges:
                    self._halo(*ex)
        inner()
        if exchanges:
            main.wait_stream(side)
        outer()

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

    def _fused_pre(self, l: int, fc, crows: int, exchanges):
        """nu1 sweeps + residual + full weighting in one pass (cycle.py:211-213)
        into fc (crows local coarse rows), after / overlapped with `exchanges`."""
        s = self.strips[l - 1]
        u, uo, zero = s.v[s.cur], s.v[s.cur ^ 1], s.vzero
        args = (u, s.f, uo, fc, s.ny, s.m, crows, s.a, s.m, self.w[l - 1], self.omega, self.nu1, zero)
        win = pre_windows(s.ny, crows, self.nu1) if self.overlap else None
        self._exchange_then(
            exchanges, lambda: self.ops.pre(*args),
            None if win is None else (lambda: self.ops.pre(*args, window=win[0], hb=0)),
            None if win is None else (lambda: [self.ops.pre(*args, window=w) for w in win[1]]))
        if self.nu1 > 0:
            s.cur ^= 1
            s.vzero = False

    def _fused_post(self, l: int, vc, vc_rows: int, exchanges, vc_halo: bool):
        """v + P vc and nu2 sweeps in one pass (cycle.py:219-220)."""
        s = self.strips[l - 1]
        args = (s.v[s.cur], s.f, s.v[s.cur ^ 1], vc, s.ny, s.m, vc_rows, s.a, s.m, self.w[l - 1], self.omega,
                self.nu2, s.vzero)
        win = post_windows(s.ny, vc_rows, self.nu2, vc_halo) if self.overlap else None
        hbc = 0 if vc_halo else HALO
        self._exchange_then(
            exchanges, lambda: self.ops.post(*args),
            None if win is None else (lambda: self.ops.post(*args, window=win[0], hb=0, hbc=hbc)),
            None if win is None else (lambda: [self.ops.post(*args, window=w) for w in win[1]]))
        s.cur ^= 1
        s.vzero = False

    def _cycle(self, l: int, kappa: int):
        s = self.strips[l - 1]
        nd = self.plan.n_dist
        fused = self._fused(l)
        pending = [(s, s.f, HALO)] if s.fpend else []  # f restricted into this level by the parent
        s.fpend = False
        if fused:  # the last owned coarse row reaches nu1 + 2 fine rows below the strip
            if not s.vzero:
                pending.append((s, s.v[s.cur], self.nu1 + 2))
        else:
            for ex in pending:
                self._halo(*ex)
            self._relax(l, self.nu1)
            if not s.vzero:
                self._halo(s, s.v[s.cur], 2)
        if l < nd:  # restrict into the next distributed strip
            c = self.strips[l]
            if fused:
                self._fused_pre(l, c.f, c.ny, pending)
            else:
                self.ops.resid_restrict(s.v[s.cur], s.f, c.f, c.ny, c.m, self.w[l - 1], s.vzero)
            c.fpend = True  # exchanged by the child's first pass (overlapped with its interior rows)
            c.vzero = True
            self._cycle(l + 1, kappa)
            if kappa > 1:
                self._cycle(l + 1, kappa - 1)
            vc, vc_rows = c.v[c.cur], c.ny
            post_ex = [(c, vc, self.nu2 // 2 + 2)]
        else:  # agglomerate: all-gather the coarse rows, replicated sub-cycle
            mc = self.plan.side(l + 1)
            q0, q1 = s.a // 2, (s.b // 2 if self.rank < self.world - 1 else mc)
            maxq = max((b // 2 if r < self.world - 1 else mc) - a // 2 for r, (a, b) in enumerate(self.plan.rows[l - 1]))
            part = self.ops.zeros(maxq + 2 * HALO, self.cfull.shape[1])
            if fused:
                self._fused_pre(l, part, q1 - q0, pending)
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
            post_ex = []
        if fused:
            if not s.vzero:
                post_ex.append((s, s.v[s.cur], max(self.nu2, 1)))
            self._fused_post(l, vc, vc_rows, post_ex, vc_halo=l < nd)
        else:
            for ex in post_ex:
                self._halo(*ex)
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
        """One cycle (and optionally the norms of its result)."""
        self._graphed((k, with_norms), lambda: self._body(k, with_norms))

    def _graphed(self, key, fn):
        """Run fn(): eager on the first call per key, then captured once into
        a CUDA graph (CUDA strips, NCCL and the native coarse engine all on
        torch's stream) and replayed."""
        if self._graphs_ok and key in self._warm:
            g = self._graphs.get(key)
            if g is None:
                g = self._capture(key, fn)
            if g is not None:
                g.replay()
                self._replayed += self._key_launches.get(key, 0)
                return
        before = self._enqueued()
        fn()
        self._key_launches[key] = self._enqueued() - before
        self._warm.add(key)

    def _enqueued(self) -> int:
        return getattr(self.ops, "launches", 0) + getattr(self.coarse, "launches", 0)

    def kernels_launched(self) -> int:
        """Kernels this rank has launched so far: eager calls (counted by the
        strip ops and the coarse engine) plus graph replays (each replay counts
        the kernels its body enqueued when it ran eagerly); bench gpu_launches."""
        return self._replayed + self._enqueued()

    def _capture(self, key, fn):
        """Capture fn() into a CUDA graph; None (eager from then on, with a
        warning and `graph_fallback` set) when it does not return the strips
        to their buffer parity (a replayed graph would read the wrong buffers)
        or cannot be captured."""
        import torch
        state0 = self._host_state()
        counts0 = (getattr(self.ops, "launches", 0), getattr(self.coarse, "launches", 0))
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        why = None
        try:
            with torch.cuda.graph(g):
                fn()
        except Exception as exc:  # a backend that cannot be captured: stay eager
            why = f"capture failed: {exc!r}"
        else:
            if self._host_state() != state0:
                why = "the captured work does not return the strips to their buffer parity"
        # the capture enqueued nothing: undo what the host walk counted
        if hasattr(self.ops, "launches"):
            self.ops.launches = counts0[0]
        if hasattr(self.coarse, "launches"):
            self.coarse.launches = counts0[1]
        if why is not None:
            for st, (cur, vz) in zip(self.strips, state0):
                st.cur, st.vzero = cur, vz
            self._graphs_ok = False
            self.graph_fallback = why
            import warnings
            warnings.warn(f"distributed solver: CUDA graphs off, running eagerly ({why})")
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

    # -- device-side loops -------------------------------------------------
    def _ds_buffers(self, hist_len: int):
        """Scalars (KC_DS_* slots), reduction scratch and the history, once per
        solver (the history grows when a longer loop asks for it)."""
        if getattr(self, "_scal", None) is None:
            self._scal = self.ops.vector(DS_SLOTS)
            self._part = self.ops.vector(DS_PART)
        if getattr(self, "_hist", None) is None or self._hist.numel() < hist_len:
            self._hist = self.ops.vector(hist_len)
        return self._scal, self._part, self._hist

    def _allreduce_slots(self, scal, a: int, b: int):
        """Allreduce scal[a:b] in place (a contiguous view: one NCCL call)."""
        self.comm.allreduce_sum(scal[a:b])

    def _read_scalars(self, scal) -> list[float]:
        return [float(v) for v in scal.cpu().tolist()]

    def _scatter(self, t, full):
        """Own rows of a global finest-level host array into strip tensor t."""
        s = self.strips[0]
        rows = np.asarray(full, dtype=np.float64)[s.a:s.b]
        host = np.zeros((s.ny, t.shape[1]))
        host[:, KC_OX:KC_OX + s.m] = rows
        t[HALO:HALO + s.ny].copy_(self.ops.torch.from_numpy(host) if hasattr(self.ops, "torch") else host)

    def _gather(self, t) -> np.ndarray:
        s = self.strips[0]
        maxrows = max(b - a for a, b in self.plan.rows[0])
        buf = self.ops.zeros(maxrows, t.shape[1])
        buf[:s.ny].copy_(t[HALO:HALO + s.ny])
        parts = self.comm.allgather(buf)
        out = np.empty((s.m, s.m))
        for r, (a, b) in enumerate(self.plan.rows[0]):
            out[a:b] = parts[r][:b - a, KC_OX:KC_OX + s.m].cpu().numpy()
        return out

    def _precondition(self, k: int):
        """z = M r (krylov.py:81-86): one kappa-cycle from the zero guess on
        f = r, which lives in the finest strip's f; z is the finest v."""
        s = self.strips[0]
        self._halo(s, s.f, HALO)
        s.vzero = True
        self._cycle(1, k)
        self._materialize(s)
        return s.v[s.cur]

    def solve_standalone(self, target_reduction=1e8, max_cycles=10000, initial_guess=None, stop="error",
                         resident=False, batch: int = 8, kappa=None):
        """Distributed solve_standalone (cycle.py:303-366); every rank returns
        the same report.  The stopping test runs on the device (KC_DS_SOLVE:
        the reference's target, growth-streak and max_cycles rules): a batch
        of `batch` cycles + norms + step is one graph replay and the host
        reads the done flag once per batch; cycles a batch runs past the stop
        are discarded (the iterate at the stop is saved on the device).
        resident=True solves from the finest v/f already on the devices;
        kappa overrides the config's cycle counter."""
        if target_reduction <= 1.0:
            raise ValueError(f"target reduction must exceed 1, got {target_reduction}")
        if stop not in ("error", "residual"):
            raise ValueError(f"stop must be 'error' or 'residual', got {stop!r}")
        m = self.plan.side(1)
        s = self.strips[0]
        if not resident:
            v0 = (np.random.default_rng(self.problem.seed).random((m, m)) if initial_guess is None
                  else np.asarray(initial_guess, dtype=np.float64))
            self.set_level1("v", v0)
            self.set_level1("f", np.zeros((m, m)))
        self._materialize(s)
        scal, part, hist = self._ds_buffers(2 * (max_cycles + 1))
        if getattr(self, "_sol", None) is None:
            self._sol = self.ops.zeros(s.ny + 2 * HALO, s.f.shape[1])
        scal.zero_()
        init = np.zeros(DS_SLOTS)
        init[DS["MAXIT"]] = max_cycles
        init[DS["STOP_RESIDUAL"]] = 1.0 if stop == "residual" else 0.0
        init[DS["REDUCTION"]] = target_reduction
        scal.copy_(self.ops.torch.from_numpy(init))
        k = self.config.effective_kappa if kappa is None else min(self.n, int(kappa) if kappa != math.inf else self.n)
        e2 = DS["E2"]

        def norms_step():
            self._halo(s, s.v[s.cur], 1)
            self.ops.norms(s.v[s.cur], s.f, s.ny, s.m, self.w[0], out=scal[e2:e2 + 2])
            self._allreduce_slots(scal, e2, e2 + 2)
            self.ops.dist_step(DS_SOLVE, scal, hist)
            self.ops.copy_if(s.v[s.cur], self._sol, s.ny, s.m, scal)

        def body():
            for _ in range(batch):
                self._cycle(1, k)
                norms_step()

        stats = CycleStats.for_levels(self.n)
        t0 = time.perf_counter()
        k0 = self.kernels_launched()
        norms_step()  # cycle 0: the initial norms and target (cycle.py:333-341)
        done = self._read_scalars(scal)[DS["DONE"]] != 0.0
        while not done:
            self._graphed(("solve", k, batch, stop, hist.data_ptr()), body)
            done = self._read_scalars(scal)[DS["DONE"]] != 0.0
        sc = self._read_scalars(scal)
        it = int(sc[DS["IT"]])
        status = STATUS_NAMES[int(sc[DS["STATUS"]])]
        h = hist[: 2 * (it + 1)].cpu().numpy().reshape(-1, 2)
        wall_ms = 1e3 * (time.perf_counter() - t0)
        s.v[s.cur].copy_(self._sol)  # the iterate at the stop
        if it:
            if k not in self._stats_cache:
                st = CycleStats.for_levels(self.n)
                kappa_cycle(DryState(self.n, self.nu1, self.nu2), 1, k, st)
                self._stats_cache[k] = st
            stats.absorb(self._stats_cache[k], it)
        return {"status": status, "iterations": it, "err_hist": h[:, 0].tolist(), "res_hist": h[:, 1].tolist(),
                "stats": stats, "wall_ms": wall_ms, "gpu_launches": self.kernels_launched() - k0}

    def pcg_solve(self, f, x0=None, target_reduction=1e8, max_iterations=10000, stop="residual", batch: int = 4,
                  kappa=None, resident: bool = False, gather: bool = True):
        """Distributed pcg_solve (krylov.py:60-141) preconditioned by one
        distributed kappa-cycle (krylov.py:81-86); every rank passes the same
        host f / x0 and returns the same report.  Dot products are per-rank
        partial sums + an in-place allreduce (NCCL): p.Ap, the stop measure
        and r.z -- three per iteration.  alpha, beta, the breakdown and stop
        tests run on the device (KC_DS_PCG_*), so `batch` iterations are one
        graph replay with one host read of the done flag; iterations a batch
        runs past the stop leave x, r, p untouched.  resident=True reuses the
        f and x0 a previous call uploaded (kept on the devices; repeat solves
        without host traffic); gather=False skips collecting the solution."""
        if target_reduction <= 1.0:
            raise ValueError(f"target reduction must exceed 1, got {target_reduction}")
        if stop not in ("error", "residual"):
            raise ValueError(f"stop must be 'error' or 'residual', got {stop!r}")
        m = self.plan.side(1)
        s = self.strips[0]
        ops = self.ops
        if getattr(self, "_pcgv", None) is None:
            shape = (s.ny + 2 * HALO, s.f.shape[1])
            self._pcgv = {name: ops.zeros(*shape) for name in ("x", "p", "ap", "b", "x0")}
        V = self._pcgv
        scal, part, hist = self._ds_buffers(max_iterations + 1)
        measure_x = stop == "error"
        if not resident:
            self._scatter(V["b"], f)
            self._scatter(V["x0"], np.zeros((m, m)) if x0 is None else x0)
        V["x"].copy_(V["x0"])
        self._halo(s, V["x"], 1)
        ops.residual(V["x"], V["b"], s.f, s.ny, s.m, self.w[0])  # r = f - A x, kept in the finest f
        scal.zero_()
        meas = DS["MEAS"]
        a, b = (V["x"], V["x"]) if measure_x else (s.f, s.f)
        ops.dot(a, b, s.ny, s.m, part, scal, meas)
        self._allreduce_slots(scal, meas, meas + 1)
        stats = CycleStats.for_levels(self.n)
        k = self.config.effective_kappa if kappa is None else min(self.n, int(kappa) if kappa != math.inf else self.n)
        t0 = time.perf_counter()
        norm0 = math.sqrt(self._read_scalars(scal)[meas])
        target = norm0 / target_reduction
        init = np.zeros(DS_SLOTS)
        init[DS["TARGET"]], init[DS["MAXIT"]] = target, max_iterations
        scal.copy_(ops.torch.from_numpy(init))
        hist[:1].fill_(norm0)
        napp = 0
        status, it = "max_cycles", 0
        if norm0 <= target:
            status = "converged"
        else:
            z = self._precondition(k)
            napp += 1
            ops.dot(s.f, z, s.ny, s.m, part, scal, DS["RZN"])
            self._allreduce_slots(scal, DS["RZN"], DS["RZN"] + 1)
            ops.dist_step(DS_PCG_RZ0, scal, hist)
            V["p"].copy_(z)
            sc = self._read_scalars(scal)
            if sc[DS["DONE"]] != 0.0:
                status = STATUS_NAMES[int(sc[DS["STATUS"]])]
            elif max_iterations > 0:
                rzn = DS["RZN"]

                def iteration():
                    self._halo(s, V["p"], 1)
                    ops.apply_dot(V["p"], V["ap"], s.ny, s.m, self.w[0], part, scal, DS["PAP"])
                    self._allreduce_slots(scal, DS["PAP"], DS["PAP"] + 1)
                    ops.dist_step(DS_PCG_PAP, scal, hist)
                    ops.pcg_update_xr(V["x"], s.f, V["p"], V["ap"], s.ny, s.m, measure_x, part, scal)
                    self._allreduce_slots(scal, meas, meas + 1)
                    ops.dist_step(DS_PCG_MEAS, scal, hist)
                    zz = self._precondition(k)
                    ops.dot(s.f, zz, s.ny, s.m, part, scal, rzn)
                    self._allreduce_slots(scal, rzn, rzn + 1)
                    ops.dist_step(DS_PCG_RZ, scal, hist)
                    ops.pcg_update_p(V["p"], zz, s.ny, s.m, scal)

                def body():
                    for _ in range(batch):
                        iteration()

                done = False
                while not done:
                    self._graphed(("pcg", k, batch, measure_x, hist.data_ptr()), body)
                    done = self._read_scalars(scal)[DS["DONE"]] != 0.0
                sc = self._read_scalars(scal)
                it = int(sc[DS["IT"]])
                status = STATUS_NAMES[int(sc[DS["STATUS"]])]
                # applications that counted: one per iteration that reached its z = M r
                napp += it if status != "converged" and not (status == "breakdown" and
                                                              math.isnan(float(hist[it]))) else it - 1
        wall_ms = 1e3 * (time.perf_counter() - t0)
        hv = hist[: it + 1].cpu().numpy().tolist()
        if status == "breakdown" and it > 0 and math.isnan(hv[it]):
            hv = hv[:it]  # a p.Ap breakdown took no measure at that step
        if napp:
            if k not in self._stats_cache:
                st = CycleStats.for_levels(self.n)
                kappa_cycle(DryState(self.n, self.nu1, self.nu2), 1, k, st)
                self._stats_cache[k] = st
            stats.absorb(self._stats_cache[k], napp)
        return {"status": status, "iterations": it, "hist": hv, "stats": stats, "wall_ms": wall_ms,
                "solution": self._gather(V["x"]) if gather else None, "preconditioner_applications": napp}
