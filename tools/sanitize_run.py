"""Small-grid workload covering every kernel class, for compute-sanitizer
(memcheck / racecheck / synccheck; one tool per run):

  2D  all 7 smoother kinds on 33^2 and 66x34 (warp-local bins, point kernel),
      tweed / wireframe / zebra_x / zebra_y on 257^2 with TMG_CHUNK=1 (legs
      and rings spanning CTAs: cluster bins with DSMEM PCR, split cluster
      barriers), V-cycles of every hybrid layout, the while-graph solve loop;
  3D  wireframe and tweed cubes 16^3 / 32^3 (ring, frame and hub wblock
      kernels, hybrid views via TMG_HYB_MIN=4, 64-thread edges via
      TMG_FORCE_TE=64), the cube V-cycle and solve loop.

usage: compute-sanitizer --tool racecheck python tools/sanitize_run.py [2d|3d|all]
The environment knobs are read once per process, so the cluster and wide-edge
cases run in child processes (each under the same sanitizer, --target-processes all).
"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_2d(sizes=((32, 32), (66, 34)), kinds=None):
    import torch

    from paper_2110_08389_b200 import grid, mgcycle, smoothers, stencil
    from paper_2110_08389_b200.rng import Lcg64
    kinds = kinds or smoothers.KINDS
    for nx, ny in sizes:
        x = grid.make_coords("wall", nx, 1.0, 2.0)
        y = grid.make_coords("wall", ny, 1.0, 2.0)
        st = stencil.assemble(x, y)
        f = np.zeros((nx + 1, ny + 1))
        f[1:-1, 1:-1] = Lcg64(5).fill((nx - 1, ny - 1)) - 0.5
        fd = torch.from_numpy(f).cuda()
        for kind in kinds:
            u = torch.zeros_like(fd)
            smoothers.sweep(kind, st, smoothers.PlanBundle(nx, ny), u, fd)
            h = grid.build_hierarchy(x, y)
            cfg = mgcycle.CycleConfig(smoother=kind, nu1=2, nu2=2, tol=1e-8, max_cycles=3)
            mgcycle.v_cycle(h, cfg, u, fd)
            mgcycle.solve(h, cfg, fd)
        torch.cuda.synchronize()
        print(f"2d {nx}x{ny} ok", flush=True)


def run_3d(ns=(16, 32)):
    import torch

    from paper_2110_08389_b200 import configs, cube, grid, mgcycle
    for n in ns:
        for scheme in ("wireframe", "tweed"):
            x = configs.sinh_centre(n, 1.0, 3.0) if scheme == "wireframe" else \
                grid.make_tanh_wall(n, 1.0, 3.0)
            h = cube.CubeHierarchy(x, scheme=scheme)
            f = cube.config5_rhs(n)
            u = torch.zeros_like(f)
            cube.sweep(h, u, f)
            cfg = mgcycle.CycleConfig(smoother=scheme, nu1=2, nu2=2, tol=1e-8, max_cycles=3)
            cube.v_cycle(h, cfg, u, f)
            cube.solve(h, cfg, f)
            torch.cuda.synchronize()
            print(f"3d {scheme} {n} ok", flush=True)


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what == "child2d":
        run_2d(sizes=((256, 256),), kinds=("tweed", "wireframe", "zebra_x", "zebra_y"))
        return
    if what == "child3d":
        run_3d(ns=(16, 32))
        return
    if what in ("2d", "all"):
        run_2d()
        env = dict(os.environ, TMG_CHUNK="1")
        subprocess.run([sys.executable, __file__, "child2d"], env=env, check=True)
    if what in ("3d", "all"):
        run_3d()
        env = dict(os.environ, TMG_HYB_MIN="4", TMG_FORCE_TE="64")
        subprocess.run([sys.executable, __file__, "child3d"], env=env, check=True)
    print("sanitize workload done", flush=True)


if __name__ == "__main__":
    main()
