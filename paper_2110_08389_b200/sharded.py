"""Sharded V-cycle: one process per GPU, the fine levels split between ranks
(DESIGN.md §6).

Decomposition.  Every smoother that shards groups its blocks into a chain
of *sharding groups* (tmg_layout.h ``point_group``):

==============  ==========================  ====================
kind            group of interior (i, j)    blocks of a group
==============  ==========================  ====================
tweed           max(i', j')                 4 L-shells / cross / strip line
wireframe       min(i', j')                 one ring (or the centre)
zebra_x         j                           one x-line
zebra_y         i                           one y-line
checkerboard    i                           the points of column i
==============  ==========================  ====================

with i' = min(i, nx - i), j' = min(j, ny - j).  Every block lies inside one
group, a point's stencil neighbours lie in groups g-1..g+1, and coarse group
G is fine group 2G.  A rank owns a contiguous group range, so no block ever
crosses ranks: there is no partitioned line solve, only halo exchange of
whole groups with the two neighbouring ranks.  This replaces the i-slab +
SPIKE plan sketched in SURVEY.md §8(e) -- tweed legs and wireframe edges
that would cross a slab never cross a group boundary -- and keeps the
sharded result bit-identical to the single-GPU one (the same block solves
on the same inputs).

Per V-cycle level (mgcycle.py:89-104 with smoothers.py:139-150 split):

* sweep: each colour stage runs on the rank's blocks, then the ranks swap
  ``HALO`` = 2 groups of u with each neighbour;
* residual + restriction: computed for the rank's coarse groups and their
  halo only (tiles outside skip); the coarse points a rank owns only read
  fine defects within one group of its range, which the width-2 u halo and
  width-2 f halo keep exact; the coarse f halo is then swapped;
* prolongation + correction on the rank's fine groups, then a u halo swap;
* residual norm: max over the owned groups, then an all-reduce (MAX);
* coarse levels: once a rank would own fewer than ``min_groups`` groups the
  ranks all-gather the coarse right-hand side and every rank runs the rest
  of the cycle redundantly on its own GPU (no scatter is needed).

Arithmetic is entirely in the sm_100a library (``tmg_session_*`` entry
points); torch.distributed (NCCL between GPUs, gloo for the CPU tests)
moves the halo buffers.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _device, _lib

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover
    torch = None
    dist = None

SHARDABLE = ("checkerboard", "zebra_x", "zebra_y", "tweed", "wireframe")
HALO = 2


# ---------------------------------------------------------------------------
# partition (host logic)

def group_count(kind: str, nx: int, ny: int) -> int:
    return int(_lib.lib().tmg_group_count(_lib.KIND_IDS[kind], nx, ny))


def group_sizes(kind: str, nx: int, ny: int) -> np.ndarray:
    """sizes[g] = interior points of group g (index 0 unused)."""
    L = _lib.lib()
    need = L.tmg_group_sizes(_lib.KIND_IDS[kind], nx, ny, None, 0)
    if need < 0:
        raise ValueError(L.tmg_last_error().decode())
    out = np.zeros(need, dtype=np.int64)
    L.tmg_group_sizes(_lib.KIND_IDS[kind], nx, ny, ctypes.c_void_p(out.ctypes.data), need)
    return out


def group_offsets(kind: str, nx: int, ny: int, g0: int, g1: int) -> np.ndarray:
    """Encoded work-field positions of the points of groups [g0, g1)."""
    L = _lib.lib()
    kid = _lib.KIND_IDS[kind]
    n = L.tmg_group_offsets(kid, nx, ny, g0, g1, None, 0)
    if n < 0:
        raise ValueError(L.tmg_last_error().decode())
    out = np.zeros(max(n, 1), dtype=np.int64)
    L.tmg_group_offsets(kid, nx, ny, g0, g1, ctypes.c_void_p(out.ctypes.data), n)
    return out[:n]


def balanced_bounds(sizes: np.ndarray, world: int) -> list:
    """Split groups 1..G into `world` contiguous ranges of nearly equal point
    counts; returns bounds b with rank r owning [b[r], b[r+1])."""
    G = len(sizes) - 1
    if world < 1 or G < world:
        raise ValueError(f"cannot split {G} groups between {world} ranks")
    cum = np.cumsum(sizes[1:])  # cum[g-1] = points in groups 1..g
    total = cum[-1]
    b = [1]
    for r in range(1, world):
        g = int(np.searchsorted(cum, total * r / world)) + 1  # first group reaching the target
        b.append(min(max(g + 1, b[-1] + 1), G + 1 - (world - r)))
    b.append(G + 1)
    return b


def coarse_bounds(bounds: list, gc: int) -> list:
    """Nested coarse ranges: coarse group G belongs to the owner of fine
    group 2G, so rank r owns [ceil(b_r / 2), ceil(b_{r+1} / 2))."""
    cb = [min(max((b + 1) // 2, 1), gc + 1) for b in bounds]
    cb[0], cb[-1] = 1, gc + 1
    return cb


@dataclass
class ShardPlan:
    """Group ranges of every rank on the sharded levels 0..nshard-1 and on
    the first replicated level (whose owned points are all-gathered)."""

    kind: str
    dims: list
    world: int
    bounds: list = field(default_factory=list)  # per level in 0..min(nshard, L-1)
    nshard: int = 0

    @classmethod
    def build(cls, kind, dims, world, sizes_fn=None, min_groups=4):
        if kind not in SHARDABLE:
            raise ValueError(f"smoother {kind!r} does not shard (pair kinds alternate "
                             f"two decompositions); use one of {SHARDABLE}")
        sizes_fn = sizes_fn or group_sizes
        p = cls(kind, list(dims), world)
        L = len(dims)
        if world == 1 or L == 1:
            return p
        nx, ny = dims[0]
        sizes = sizes_fn(kind, nx, ny)
        if len(sizes) - 1 < world * min_groups:
            return p
        b = balanced_bounds(sizes, world)
        for lvl in range(L):
            p.bounds.append(b)
            owned = min(b[r + 1] - b[r] for r in range(world))
            if lvl == L - 1 or owned < min_groups:
                break
            p.nshard = lvl + 1
            if lvl + 1 < L:
                nxc, nyc = dims[lvl + 1]
                b = coarse_bounds(b, len(sizes_fn(kind, nxc, nyc)) - 1)
        if p.nshard == 0:
            p.bounds = []
        else:
            p.bounds = p.bounds[:p.nshard + 1]
        return p

    def own(self, level: int, rank: int):
        b = self.bounds[level]
        return b[rank], b[rank + 1]

    def halo(self, level: int, rank: int):
        """[(peer, send range, recv range)] for the two neighbours."""
        b = self.bounds[level]
        G = b[-1] - 1
        g0, g1 = b[rank], b[rank + 1]
        out = []
        if rank > 0:
            out.append((rank - 1, (g0, min(g0 + HALO, g1)), (max(g0 - HALO, 1), g0)))
        if rank < self.world - 1:
            out.append((rank + 1, (max(g1 - HALO, g0), g1), (g1, min(g1 + HALO, G + 1))))
        return out

    @property
    def tail_level(self) -> int:
        """First replicated level (len(dims) when every level shards)."""
        return self.nshard


# ---------------------------------------------------------------------------
# communication

class Comm:
    """torch.distributed plumbing: halo swaps, all-gather, max all-reduce.
    Works on CUDA tensors with NCCL and on CPU tensors (or CUDA tensors
    staged through the host) with gloo."""

    def __init__(self, group=None):
        self.group = group
        if dist is not None and dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
            self.backend = str(dist.get_backend(group))
        else:
            self.rank, self.world, self.backend = 0, 1, "none"

    def _wire(self, t):
        return t.cpu() if (self.backend == "gloo" and t.is_cuda) else t

    def exchange(self, pairs):
        """pairs: [(peer, send tensor, recv tensor)]; all posted together."""
        if self.world == 1 or not pairs:
            return
        ops, back = [], []
        for peer, snd, rcv in pairs:
            ws = self._wire(snd)
            wr = self._wire(rcv) if rcv is not None else None
            if ws.numel():
                ops.append(dist.P2POp(dist.isend, ws, peer, self.group))
            if wr is not None and wr.numel():
                ops.append(dist.P2POp(dist.irecv, wr, peer, self.group))
                if wr is not rcv:
                    back.append((wr, rcv))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for wr, rcv in back:
            rcv.copy_(wr)

    def allgather(self, t, counts):
        """Concatenate every rank's 1D tensor (lengths `counts`) in rank order."""
        if self.world == 1:
            return t
        m = max(max(counts), 1)
        buf = torch.zeros(m, dtype=t.dtype, device=t.device)
        buf[:t.numel()] = t
        wb = self._wire(buf)
        outs = [torch.empty_like(wb) for _ in range(self.world)]
        dist.all_gather(outs, wb, group=self.group)
        cat = torch.cat([o[:c] for o, c in zip(outs, counts)])
        return cat.to(t.device)

    def allreduce_max(self, values, device):
        """Elementwise max of a list of floats over the ranks."""
        if self.world == 1:
            return list(values)
        t = torch.tensor(values, dtype=torch.float64, device=device)
        wt = self._wire(t)
        dist.all_reduce(wt, op=dist.ReduceOp.MAX, group=self.group)
        return [float(x) for x in wt.cpu().tolist()]


# ---------------------------------------------------------------------------
# local operators of one rank (the product path: the sm_100a library)

class NativeShardOps:
    """One rank's work fields live in the native hierarchy session (hybrid
    N/T layout); every operator below is one C-ABI call on the current
    torch stream."""

    device = "cuda"

    def __init__(self, h, kind, restriction="full", nu1=2, nu2=2):
        _device.require_cuda()
        self.h = h
        self.kind = kind
        self.kid = _lib.KIND_IDS[kind]
        self.full = 1 if restriction == "full" else 0
        self.nu1, self.nu2 = int(nu1), int(nu2)
        self.native = h.native()
        self.L = _lib.lib()
        self.dims = [(lv.nx, lv.ny) for lv in h.levels]

    def _s(self):
        return _device.stream_handle()

    def group_sizes(self, kind, nx, ny):
        return group_sizes(kind, nx, ny)

    def offsets(self, level, g0, g1):
        nx, ny = self.dims[level]
        return torch.from_numpy(group_offsets(self.kind, nx, ny, g0, g1)).to("cuda")

    def buffer(self, n):
        return torch.empty(n, dtype=torch.float64, device="cuda")

    def load(self, u, f):
        _lib.check(self.L.tmg_session_load(self.native, self.kid, _device.ptr(u),
                                           _device.ptr(f), self._s()))

    def store(self, u):
        _lib.check(self.L.tmg_session_store(self.native, _device.ptr(u), self._s()))

    def gather(self, level, which, idx, out):
        _lib.check(self.L.tmg_session_gather(self.native, level, which, _device.ptr(idx),
                                             idx.numel(), _device.ptr(out), self._s()))

    def scatter(self, level, which, idx, buf):
        _lib.check(self.L.tmg_session_scatter(self.native, level, which, _device.ptr(idx),
                                              idx.numel(), _device.ptr(buf), self._s()))

    def sweep(self, level, red, g0, g1):
        _lib.check(self.L.tmg_session_sweep_part(self.native, level, self.kid, int(red), g0, g1,
                                                 self._s()))

    def restrict(self, level, groups=None):
        """f[level+1] = R(f - Lu), u[level+1] = 0; groups = (g0, g1): only the
        coarse points of those sharding groups (one rank's share + halo)."""
        if groups is None:
            _lib.check(self.L.tmg_session_restrict(self.native, level, self.full, self._s()))
        else:
            _lib.check(self.L.tmg_session_restrict_part(self.native, level, self.full, self.kid,
                                                        int(groups[0]), int(groups[1]),
                                                        self._s()))

    def prolong(self, level, groups=None):
        """u[level] += P u[level+1]; groups = (g0, g1): only those fine groups."""
        if groups is None:
            _lib.check(self.L.tmg_session_prolong(self.native, level, self._s()))
        else:
            _lib.check(self.L.tmg_session_prolong_part(self.native, level, self.kid,
                                                       int(groups[0]), int(groups[1]),
                                                       self._s()))

    def tail(self, level):
        _lib.check(self.L.tmg_session_tail(self.native, level, self.kid, self.full, self.nu1,
                                           self.nu2, self._s()))

    def norm(self, g0, g1):
        """(owned max-norm of the finest defect, pivot error message or None)."""
        out = ctypes.c_double()
        st = self.L.tmg_session_norm_part(self.native, self.kid, g0, g1, ctypes.byref(out),
                                          self._s())
        if st == _lib.TMG_SINGULAR:
            return float("nan"), self.L.tmg_last_error().decode()
        _lib.check(st)
        return out.value, None


# ---------------------------------------------------------------------------
# driver

class ShardedSolver:
    """mgcycle.solve / v_cycle with the fine levels split between ranks.
    Every rank passes the full f (and g); every rank gets the full u."""

    def __init__(self, h, cfg, comm: Comm | None = None, ops=None, min_groups: int = 4):
        if cfg.smoother not in SHARDABLE:
            raise ValueError(f"smoother {cfg.smoother!r} does not shard; use one of {SHARDABLE}")
        self.h, self.cfg = h, cfg
        self.comm = comm or Comm()
        self.ops = ops or NativeShardOps(h, cfg.smoother, cfg.restriction, cfg.nu1, cfg.nu2)
        self.dims = list(self.ops.dims)  # per level (nx, ny); (n, n) for cubes
        self.plan = ShardPlan.build(cfg.smoother, self.dims, self.comm.world,
                                    sizes_fn=self.ops.group_sizes, min_groups=min_groups)
        r = self.comm.rank
        self.exchanges = 0
        # per level: both sides' send / receive offsets concatenated, so that a
        # swap is one gather kernel, the exchange and one scatter kernel; each
        # side's message is a view of the joint buffer
        self._halo = []
        for lvl in range(self.plan.nshard):
            peers, sis, ris = [], [], []
            for peer, (s0, s1), (r0, r1) in self.plan.halo(lvl, r):
                peers.append(peer)
                sis.append(self.ops.offsets(lvl, s0, s1))
                ris.append(self.ops.offsets(lvl, r0, r1))
            if not peers:
                self._halo.append(None)
                continue
            si, ri = torch.cat(sis), torch.cat(ris)
            sb, rb = self.ops.buffer(si.numel()), self.ops.buffer(ri.numel())
            pairs, so, ro = [], 0, 0
            for peer, a, b in zip(peers, sis, ris):
                pairs.append((peer, sb[so:so + a.numel()], rb[ro:ro + b.numel()]))
                so += a.numel()
                ro += b.numel()
            self._halo.append((si, ri, sb, rb, pairs))
        self._gathers = {}
        if self.comm.world > 1:
            # a collective before the first batched send/recv of the group
            # (NCCL requires the first P2P batch to follow one)
            self.comm.allreduce_max([0.0], self.ops.device)

    # -- plumbing ---------------------------------------------------------
    def _swap(self, level, which):
        halo = self._halo[level]
        if halo is not None:
            si, ri, sb, rb, pairs = halo
            self.ops.gather(level, which, si, sb)
            self.comm.exchange(pairs)
            self.ops.scatter(level, which, ri, rb)
        self.exchanges += 1

    def _gather_lists(self, level):
        """(my owned offsets, all ranks' owned offsets in rank order, counts)."""
        if level not in self._gathers:
            b = self.plan.bounds[level]
            lists = [self.ops.offsets(level, b[k], b[k + 1]) for k in range(self.comm.world)]
            counts = [int(x.numel()) for x in lists]
            self._gathers[level] = (lists[self.comm.rank], torch.cat(lists), counts)
        return self._gathers[level]

    def _allgather_field(self, level, which):
        mine, every, counts = self._gather_lists(level)
        buf = self.ops.buffer(mine.numel())
        self.ops.gather(level, which, mine, buf)
        allv = self.comm.allgather(buf, counts)
        self.ops.scatter(level, which, every, allv)

    # -- cycle ------------------------------------------------------------
    def _smooth(self, level, nu):
        g0, g1 = self.plan.own(level, self.comm.rank)
        for _ in range(nu):
            for red in (1, 0):
                self.ops.sweep(level, red, g0, g1)
                self._swap(level, 0)

    def _cycle(self, level):
        if level == self.plan.tail_level:
            self.ops.tail(level)
            return
        self._smooth(level, self.cfg.nu1)
        if level + 1 < self.plan.nshard:
            # the rank's coarse groups and their halo only: the owned points
            # read fine defects inside the width-2 fine halo, the halo's f is
            # swapped right after and its u must be the zero initial guess
            g0, g1 = self.plan.own(level + 1, self.comm.rank)
            G = self.plan.bounds[level + 1][-1] - 1
            self.ops.restrict(level, (max(g0 - HALO, 1), min(g1 + HALO, G + 1)))
            self._swap(level + 1, 1)
        else:  # the replicated tail needs every coarse point (u = 0 everywhere)
            self.ops.restrict(level)
            self._allgather_field(level + 1, 1)
        self._cycle(level + 1)
        self.ops.prolong(level, self.plan.own(level, self.comm.rank))
        self._swap(level, 0)
        self._smooth(level, self.cfg.nu2)

    def v_cycle(self):
        """One V-cycle on the loaded session."""
        if self.plan.nshard == 0:
            self.ops.tail(0)
        else:
            self._cycle(0)

    def norm(self):
        if self.plan.nshard == 0:
            G = len(self.ops.group_sizes(self.cfg.smoother, *self.dims[0])) - 1
            g0, g1 = 1, G + 1
        else:
            g0, g1 = self.plan.own(0, self.comm.rank)
        v, err = self.ops.norm(g0, g1)
        bad = 1.0 if err else 0.0
        v = v if np.isfinite(v) else float("inf")
        v, bad = self.comm.allreduce_max([v, bad], self.ops.device)
        if bad:
            from .tridiag import SingularSystemError
            raise SingularSystemError(err or "zero pivot on another rank")
        return v

    def load(self, u, f):
        self.ops.load(u, f)

    def store(self, u):
        if self.plan.nshard > 0:
            self._allgather_field(0, 0)
        self.ops.store(u)

    def solve(self, f, g=None):
        """V-cycles from u = 0 (boundary from g) until max|f - Lu| <= tol*d0, a
        non-finite defect or max_cycles (mgcycle.py:107-139)."""
        from .mgcycle import CycleReport
        cfg = self.cfg
        want = self.dims[0][0] + 1, self.dims[0][1] + 1
        if tuple(f.shape) != want:
            raise ValueError(f"field shape {tuple(f.shape)} does not match grid {want}")
        host = isinstance(f, np.ndarray)
        if self.ops.device == "cuda":
            fd = _device.to_device(f)
            u = torch.zeros(want, dtype=torch.float64, device="cuda")
        else:
            fd = np.ascontiguousarray(f, dtype=np.float64)
            u = np.zeros(want)
        if g is not None:
            gd = _device.to_device(g) if self.ops.device == "cuda" else np.asarray(g)
            u[0, :], u[-1, :], u[:, 0], u[:, -1] = gd[0, :], gd[-1, :], gd[:, 0], gd[:, -1]
        self.load(u, fd)
        rep = CycleReport()
        d0 = self.norm()
        rep.defect_norms.append(d0)
        if d0 == 0.0:
            rep.converged = True
        else:
            for cycle in range(1, cfg.max_cycles + 1):
                self.v_cycle()
                dn = self.norm()
                rep.defect_norms.append(dn)
                rep.relaxations.append(cycle * cfg.relaxations_per_cycle)
                rep.cycles = cycle
                if not np.isfinite(dn):
                    break
                if dn <= cfg.tol * d0:
                    rep.converged = True
                    break
        self.store(u)
        if host and self.ops.device == "cuda":
            u = u.cpu().numpy()
        return u, rep


def solve(h, cfg, f, g=None, comm: Comm | None = None):
    """Sharded counterpart of mgcycle.solve over the initialised process group."""
    return ShardedSolver(h, cfg, comm).solve(f, g)
