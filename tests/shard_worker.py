"""Worker of the multi-process sharded-solve tests (tests/test_sharded.py).

Launched as ``torchrun --nproc-per-node W --master-addr 127.0.0.1 ...
tests/shard_worker.py --ops oracle|native --kind K --nx N --out DIR``.
Each rank runs paper_2110_08389_b200.sharded.ShardedSolver over a gloo
process group and writes its u, its defect norms and the exchange count to
DIR/rank{r}.npz.

``--ops oracle`` is test infrastructure: the rank-local operators are the
CPU oracle (OracleShardOps below), so the partition, the halo protocol and
the replicated tail are checked on CPU against the single-domain oracle.
``--ops native`` runs the product path (NativeShardOps, the sm_100a library)
with the halo buffers staged through the host for gloo.
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


class OracleShardOps:
    """Rank-local operators on numpy fields in C order (the CPU oracle)."""

    device = "cpu"

    def __init__(self, oh, kind, restriction, nu1, nu2):
        from oracle import oracle
        self.o = oracle
        self.oh, self.kind, self.restriction = oh, kind, restriction
        self.nu1, self.nu2 = nu1, nu2
        self.st = oh.stencils
        self.dims = [(len(s[0]) - 1, len(s[2]) - 1) for s in self.st]
        self.U = [np.zeros((nx + 1, ny + 1)) for nx, ny in self.dims]
        self.F = [np.zeros((nx + 1, ny + 1)) for nx, ny in self.dims]
        self._gm = {}

    def _gmap(self, nx, ny):
        if (nx, ny) not in self._gm:
            self._gm[(nx, ny)] = self.o.group_map(self.kind, nx, ny)
        return self._gm[(nx, ny)]

    def group_sizes(self, kind, nx, ny):
        gm = self._gmap(nx, ny)
        return np.bincount(gm[1:-1, 1:-1].ravel(), minlength=gm.max() + 1).astype(np.int64)

    def offsets(self, level, g0, g1):
        gm = self._gmap(*self.dims[level])
        idx = np.flatnonzero((gm >= g0) & (gm < g1))
        return torch.from_numpy(2 * idx.astype(np.int64))

    def buffer(self, n):
        return torch.empty(n, dtype=torch.float64)

    def load(self, u, f):
        self.U[0][...] = u
        self.F[0][...] = f

    def store(self, u):
        u[...] = self.U[0]

    def _arr(self, level, which):
        return (self.F if which else self.U)[level].reshape(-1)

    def gather(self, level, which, idx, out):
        out.copy_(torch.from_numpy(self._arr(level, which)[idx.numpy() >> 1]))

    def scatter(self, level, which, idx, buf):
        self._arr(level, which)[idx.numpy() >> 1] = buf.numpy()

    def sweep(self, level, red, g0, g1):
        self.o.sweep_part(self.kind, self.st[level], self.U[level], self.F[level], red, g0, g1)

    def restrict(self, level, groups=None):  # whole level (groups: a rank's share)
        d = self.o.defect(self.st[level], self.U[level], self.F[level])
        self.F[level + 1][...] = self.o.restrict(self.restriction, d)
        self.U[level + 1][...] = 0.0

    def prolong(self, level, groups=None):
        self.o.prolong_add(self.U[level + 1], self.U[level])

    def tail(self, level):
        self.o._v_cycle(self.oh, self.kind, self.restriction, self.nu1, self.nu2, level,
                        self.U[level], self.F[level], 1)

    def norm(self, g0, g1):
        d = np.abs(self.o.defect(self.st[0], self.U[0], self.F[0]))
        gm = self._gmap(*self.dims[0])
        m = (gm >= g0) & (gm < g1)
        return (float(d[m].max()) if m.any() else 0.0), None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", choices=("oracle", "native"), default="oracle")
    ap.add_argument("--kind", default="tweed")
    ap.add_argument("--nx", type=int, default=64)
    ap.add_argument("--ny", type=int, default=0)
    ap.add_argument("--restriction", default="full")
    ap.add_argument("--max-cycles", type=int, default=50)
    ap.add_argument("--min-groups", type=int, default=4)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()

    dist.init_process_group("gloo")
    rank = dist.get_rank()
    from oracle import oracle
    from paper_2110_08389_b200 import grid, mgcycle, sharded

    nx, ny = args.nx, args.ny or args.nx
    x, y = grid.make_coords("wall", nx, 1.0, 3.0), grid.make_coords("wall", ny, 2.0, 2.0)
    h = grid.build_hierarchy(x, y)
    cfg = mgcycle.CycleConfig(smoother=args.kind, restriction=args.restriction,
                              max_cycles=args.max_cycles)
    f = mgcycle.random_rhs(nx, ny, 7)
    comm = sharded.Comm()
    if args.ops == "oracle":
        oh = oracle.Hierarchy(x.values, y.values)
        ops = OracleShardOps(oh, args.kind, args.restriction, cfg.nu1, cfg.nu2)
    else:
        torch.cuda.set_device(0)
        ops = sharded.NativeShardOps(h, args.kind, args.restriction, cfg.nu1, cfg.nu2)
    solver = sharded.ShardedSolver(h, cfg, comm=comm, ops=ops, min_groups=args.min_groups)
    u, rep = solver.solve(f)
    u = u.cpu().numpy() if isinstance(u, torch.Tensor) else u
    np.savez(os.path.join(args.out, f"rank{rank}.npz"), u=u,
             norms=np.array(rep.defect_norms), cycles=rep.cycles, converged=rep.converged,
             exchanges=solver.exchanges, nshard=solver.plan.nshard)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
