"""One (or a few) 3D sweeps on a cube, for ncu captures:
cube_sweep_once.py n tweed|wireframe [reps] [session]  (session: the loaded
session's sweeps, on the hybrid views of the 3D wireframe)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08389_b200 import _lib, configs, cube, grid  # noqa: E402

n = int(sys.argv[1])
scheme = sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if scheme == "tweed":
    h = cube.CubeHierarchy(grid.make_tanh_wall(n, 1.0, 3.0))
    f = cube.config4_rhs(n)
else:
    h = cube.CubeHierarchy(configs.sinh_centre(n, 1.0, 3.0), scheme="wireframe")
    f = cube.config5_rhs(n)
u = torch.zeros_like(f)
L = _lib.lib()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
if len(sys.argv) > 4 and sys.argv[4] == "session":
    L.tmg_cube_load(h._h, ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(f.data_ptr()), s)
    L.tmg_cube_sweeps(h._h, reps, s)
else:
    for _ in range(reps):
        L.tmg_cube_sweep(h._h, ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(f.data_ptr()), s)
torch.cuda.synchronize()
print("done", n, scheme, reps)
