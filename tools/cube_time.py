"""Time the 3D sweep and V(2,2) cycle on a cube: cube_time.py [n] [tweed|wireframe]
(default 257^3 tweed; wireframe uses the config-5 sinh-centre grid)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08389_b200 import _lib, configs, cube, grid  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
scheme = sys.argv[2] if len(sys.argv) > 2 else "tweed"
if scheme == "tweed":
    h = cube.CubeHierarchy(grid.make_tanh_wall(n, 1.0, 3.0))
    f = cube.config4_rhs(n)
else:
    h = cube.CubeHierarchy(configs.sinh_centre(n, 1.0, 3.0), scheme="wireframe")
    f = cube.config5_rhs(n)
u = torch.zeros_like(f)
L = _lib.lib()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
st = torch.cuda.current_stream()


def ev(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


tsw = ev(lambda: L.tmg_cube_sweep(h._h, ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(f.data_ptr()), s), 10)
L.tmg_cube_load(h._h, ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(f.data_ptr()), s)
tss = ev(lambda: L.tmg_cube_sweeps(h._h, 1, s), 10)
tcy = ev(lambda: L.tmg_cube_cycles(h._h, 2, 2, 1, s), 5)
npts = (n - 1) ** 3
print(f"{scheme} n={n} blocks {h.blocks(0)} sweep {tsw:.3f} ms ({24 * npts / tsw / 1e6:.0f} GB/s alg) "
      f"session sweep {tss:.3f} ms ({24 * npts / tss / 1e6:.0f} GB/s alg) "
      f"V(2,2) {tcy:.3f} ms ({4 * h.interior_points() / tcy / 1e6:.3e} updates/s)")
