"""Session workload for ncu: load config 3 (or --n), run --cycles V-cycles
(graph) and --sweeps finest-level sweeps on the session's hybrid layout."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08389_b200 import _lib, configs, grid, mgcycle  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="config3")
p.add_argument("--n", type=int, default=None)
p.add_argument("--sweeps", type=int, default=1)
p.add_argument("--cycles", type=int, default=1)
a = p.parse_args()
w = configs.workload(a.config, n=a.n)
h = grid.build_hierarchy(w.x, w.x)
kind = _lib.KIND_IDS[w.smoother]
f = torch.from_numpy(w.rhs()).cuda()
u = torch.zeros_like(f)
L = _lib.lib()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
st = mgcycle._CycleState(h)
_lib.check(L.tmg_session_load(st.native, kind, ctypes.c_void_p(u.data_ptr()),
                              ctypes.c_void_p(f.data_ptr()), s))
if a.cycles:
    _lib.check(L.tmg_session_cycles(st.native, kind, 1, w.nu1, w.nu2, a.cycles, s))
if a.sweeps:
    _lib.check(L.tmg_session_sweeps(st.native, kind, a.sweeps, s))
v = ctypes.c_double()
_lib.check(L.tmg_session_norm(st.native, ctypes.byref(v), s))
print("done norm", v.value)
