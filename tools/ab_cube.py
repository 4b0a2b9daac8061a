"""A/B of two library builds on the 3D cube paths (raw ctypes, symbols every
build has): ab_cube.py LIB n tweed|wireframe."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2110_08389_b200 import configs, cube, grid  # noqa: E402

L = ctypes.CDLL(sys.argv[1])
n, scheme = int(sys.argv[2]), sys.argv[3]
x = grid.make_tanh_wall(n, 1.0, 3.0) if scheme == "tweed" else configs.sinh_centre(n, 1.0, 3.0)
v = np.ascontiguousarray(x.values)
h = ctypes.c_void_p()
assert L.tmg_cube_create_scheme(n, v.ctypes.data_as(ctypes.c_void_p), 0 if scheme == "tweed" else 1,
                                ctypes.byref(h)) == 0
f = cube.config4_rhs(n) if scheme == "tweed" else cube.config5_rhs(n)
u = torch.zeros_like(f)
st = torch.cuda.current_stream()
s = ctypes.c_void_p(st.cuda_stream)
P = lambda t: ctypes.c_void_p(t.data_ptr())


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


tsw = ev(lambda: L.tmg_cube_sweep(h, P(u), P(f), s), 10)
L.tmg_cube_load(h, P(u), P(f), s)
tcy = ev(lambda: L.tmg_cube_cycles(h, 2, 2, 1, s), 5)
print(f"{os.path.basename(sys.argv[1])} {scheme} n={n} natural sweep {tsw:.3f} ms V(2,2) {tcy:.3f} ms")
