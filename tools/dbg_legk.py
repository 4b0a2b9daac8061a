import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2110_08389_b200 import _lib, grid
from paper_2110_08389_b200.rng import Lcg64
from paper_2110_08389_b200.stencil import native_level
L = _lib.lib(); s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: ctypes.c_void_p(t.data_ptr())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
x = grid.make_coords("wall", n, 1.0, 4.0); y = grid.make_coords("wall", n, 1.0, 2.0); h = grid.build_hierarchy(x, y)
rng = Lcg64(11 + n)
f = np.zeros((n + 1, n + 1)); f[1:-1, 1:-1] = rng.fill((n - 1, n - 1)) - 0.5
u = np.zeros_like(f); u[1:-1, 1:-1] = rng.fill((n - 1, n - 1)) - 0.5
fd = torch.from_numpy(f).cuda(); ud = torch.from_numpy(u).cuda(); ref = ud.clone()
lv = native_level(h.finest.stencil)
for colour in (1,):
    _lib.check(L.tmg_sweep_colour(lv, 4, colour, P(ref), P(fd), s))
hn = h.native()
_lib.check(L.tmg_session_load(hn, 4, P(ud), P(fd), s))
# one red stage only: session_sweeps does full sweeps; use 1 sweep and compare both
ref2 = torch.from_numpy(u).cuda()
_lib.check(L.tmg_sweep(lv, 4, P(ref2), P(fd), s))
_lib.check(L.tmg_session_sweeps(hn, 4, 1, s))
got = torch.empty_like(ud); _lib.check(L.tmg_session_store(hn, P(got), s)); torch.cuda.synchronize()
d = (got - ref2).abs().cpu().numpy()
bad = np.argwhere(d > 1e-10 * np.abs(ref2.cpu().numpy()).max())
print("n", n, "bad points", len(bad))
bad = sorted(bad.tolist(), key=lambda ij: -d[ij[0], ij[1]])
for i, j in bad[:25]:
    ip, jp = min(i, n - i), min(j, n - j)
    print(i, j, "shell", max(ip, jp), "colour", "red" if max(ip,jp) % 2 else "black", d[i, j],
          "got", float(got[i, j]), "ref", float(ref2[i, j]), "u0", float(u[i, j]))
