"""One 3D V(2,2) cycle on the session (graph replay), for ncu launch lists:
cube_cycle_once.py n tweed|wireframe."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08389_b200 import _lib, configs, cube, grid  # noqa: E402

n, scheme = int(sys.argv[1]), sys.argv[2]
if scheme == "tweed":
    h = cube.CubeHierarchy(grid.make_tanh_wall(n, 1.0, 3.0))
    f = cube.config4_rhs(n)
else:
    h = cube.CubeHierarchy(configs.sinh_centre(n, 1.0, 3.0), scheme="wireframe")
    f = cube.config5_rhs(n)
u = torch.zeros_like(f)
L = _lib.lib()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
L.tmg_cube_load(h._h, ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(f.data_ptr()), s)
L.tmg_cube_cycles(h._h, 2, 2, 1, s)
torch.cuda.synchronize()
print("done")
