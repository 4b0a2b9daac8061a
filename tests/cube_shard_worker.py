"""Worker of the multi-process sharded cube tests (tests/test_sharded_3d.py).

Launched as ``torchrun --nproc-per-node W --master-addr 127.0.0.1 ...
tests/cube_shard_worker.py --ops oracle|native --size N --out DIR``.  Each rank
runs paper_2110_08389_b200.cube_sharded.CubeShardedSolver (3D wireframe,
shell groups) over a gloo process group and writes its u, its defect norms
and the exchange count to DIR/rank{r}.npz.

``--ops oracle`` is test infrastructure: the rank-local operators are the
CPU oracle (oracle/wire3d_oracle.c, OracleCubeShardOps below), so the shell
partition, the halo protocol and the replicated tail are checked on CPU
against the single-domain oracle.  ``--ops native`` runs the product path
(NativeCubeShardOps, the sm_100a library), halos staged through the host
for gloo.
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


class OracleCubeShardOps:
    """Rank-local cube operators on numpy fields (the CPU oracle)."""

    device = "cpu"

    def __init__(self, oh, nu1, nu2):
        from oracle import oracle3d
        self.o = oracle3d
        self.oh, self.nu1, self.nu2 = oh, nu1, nu2
        self.st = oh.stencils
        self.dims = [(len(s[0]) - 1,) * 2 for s in self.st]
        self.U = [np.zeros((n + 1,) * 3) for n, _ in self.dims]
        self.F = [np.zeros((n + 1,) * 3) for n, _ in self.dims]
        self._gm = {}

    def _gmap(self, n):
        if n not in self._gm:
            self._gm[n] = self.o.group_map(n, "wireframe")
        return self._gm[n]

    def group_sizes(self, kind, nx, ny):
        gm = self._gmap(nx)
        return np.bincount(gm[1:-1, 1:-1, 1:-1].ravel(), minlength=nx // 2 + 1).astype(np.int64)

    def offsets(self, level, g0, g1):
        gm = self._gmap(self.dims[level][0])
        return torch.from_numpy(np.flatnonzero((gm >= g0) & (gm < g1)).astype(np.int64))

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
        out.copy_(torch.from_numpy(self._arr(level, which)[idx.numpy()]))

    def scatter(self, level, which, idx, buf):
        self._arr(level, which)[idx.numpy()] = buf.numpy()

    def sweep(self, level, red, g0, g1):
        self.o.sweep_part(self.st[level], self.U[level], self.F[level], red, g0, g1)

    def restrict(self, level, groups=None):  # whole level (groups: a rank's share)
        d = self.o.defect(self.st[level], self.U[level], self.F[level])
        self.F[level + 1][...] = self.o.restrict(d)
        self.U[level + 1][...] = 0.0

    def prolong(self, level, groups=None):
        self.o.prolong_add(self.U[level + 1], self.U[level])

    def tail(self, level):
        self.o._v_cycle(self.oh, self.nu1, self.nu2, level, self.U[level], self.F[level], 1)

    def norm(self, g0, g1):
        d = np.abs(self.o.defect(self.st[0], self.U[0], self.F[0]))
        gm = self._gmap(self.dims[0][0])
        m = (gm >= g0) & (gm < g1)
        return (float(d[m].max()) if m.any() else 0.0), None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", choices=("oracle", "native"), default="oracle")
    ap.add_argument("--size", type=int, default=16)
    ap.add_argument("--max-cycles", type=int, default=6)
    ap.add_argument("--min-groups", type=int, default=2)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()

    dist.init_process_group("gloo")
    rank = dist.get_rank()
    from oracle import oracle3d
    from paper_2110_08389_b200 import configs, cube, cube_sharded, mgcycle, sharded

    n = args.size
    x = configs.sinh_centre(n, 1.0, 3.0)
    cfg = mgcycle.CycleConfig(smoother="wireframe", max_cycles=args.max_cycles)
    f = cube.config5_rhs(n, device=False)
    comm = sharded.Comm()
    if args.ops == "oracle":
        oh = oracle3d.Hierarchy3(x.values, scheme="wireframe")
        ops, h = OracleCubeShardOps(oh, cfg.nu1, cfg.nu2), None
    else:
        torch.cuda.set_device(0)
        h = cube.CubeHierarchy(x, scheme="wireframe")
        ops = cube_sharded.NativeCubeShardOps(h, cfg.nu1, cfg.nu2)
    solver = cube_sharded.CubeShardedSolver(h, cfg, comm=comm, ops=ops,
                                            min_groups=args.min_groups)
    u, rep = solver.solve(f)
    u = u.cpu().numpy() if isinstance(u, torch.Tensor) else u
    np.savez(os.path.join(args.out, f"rank{rank}.npz"), u=u,
             norms=np.array(rep.defect_norms), cycles=rep.cycles, converged=rep.converged,
             exchanges=solver.exchanges, nshard=solver.plan.nshard)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
