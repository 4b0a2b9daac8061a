"""Short deterministic workload for ncu: build config 3 (or --n), run
--sweeps finest-level sweeps and --cycles V-cycles through the graph path."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2110_08389_b200 import _lib, configs, grid, mgcycle  # noqa: E402
from paper_2110_08389_b200.stencil import native_level  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="config3")
p.add_argument("--n", type=int, default=None)
p.add_argument("--sweeps", type=int, default=2)
p.add_argument("--cycles", type=int, default=1)
p.add_argument("--kind", default=None)
a = p.parse_args()
w = configs.workload(a.config, n=a.n)
h = grid.build_hierarchy(w.x, w.x)
kind = _lib.KIND_IDS[a.kind or w.smoother]
f = torch.from_numpy(w.rhs()).cuda()
u = torch.zeros_like(f)
L = _lib.lib()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
up, fp = ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(f.data_ptr())
lv = native_level(h.finest.stencil)
for _ in range(a.sweeps):
    _lib.check(L.tmg_sweep(lv, kind, up, fp, s))
if a.cycles:
    st = mgcycle._CycleState(h)
    _lib.check(L.tmg_vcycle_graph(st.native, kind, 1, w.nu1, w.nu2, up, fp, a.cycles, s))
torch.cuda.synchronize()
_lib.check(L.tmg_level_check(lv, s))
print("done", float(u.abs().max()))
