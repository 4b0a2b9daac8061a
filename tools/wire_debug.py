"""Per-block-kind error of one device 3D wireframe sweep against the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2110_08389_b200 import configs, cube
from oracle import oracle3d as o3
n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
x = configs.sinh_centre(n, 1.0, 3.0)
h = cube.CubeHierarchy(x, scheme="wireframe")
rng = np.random.default_rng(5)
u = np.zeros((n + 1,) * 3)
u[1:-1, 1:-1, 1:-1] = rng.standard_normal((n - 1,) * 3)
f = rng.standard_normal((n + 1,) * 3)
ug = u.copy()
cube.sweep(h, ug, f)
uo = u.copy()
o3.sweep(o3.assemble3(x.values, x.values, x.values), uo, f, scheme="wireframe")
ii, jj, kk, blk, red = o3.layout_dump(n, "wireframe")
m = lambda v: np.minimum(v, n - v)
for (i, j, k) in zip(ii, jj, kk):
    e = abs(ug[i, j, k] - uo[i, j, k])
    if e > 1e-12:
        s = sorted((m(i), m(j), m(k)))
        print((i, j, k), "frame" if s[0] == s[1] else "ring", s, f"{ug[i,j,k]:.6f} {uo[i,j,k]:.6f}")
print("max err", np.abs(ug - uo).max())
