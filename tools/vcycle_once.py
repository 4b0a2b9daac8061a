"""Load the config-3 session, warm up, then run ONE V(2,2) cycle (for ncu launch lists)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08389_b200 import _lib, configs, grid, mgcycle

w = configs.workload(sys.argv[1] if len(sys.argv) > 1 else "config3")
h = grid.build_hierarchy(w.x, w.x)
f = torch.from_numpy(w.rhs()).cuda()
u = torch.zeros_like(f)
L = _lib.lib()
st = mgcycle._CycleState(h)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
kind = 4 if w.smoother == "tweed" else 5
_lib.check(L.tmg_session_load(st.native, kind, ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(f.data_ptr()), s))
_lib.check(L.tmg_session_cycles(st.native, kind, 1, 2, 2, 1, s))
torch.cuda.synchronize()
_lib.check(L.tmg_session_cycles(st.native, kind, 1, 2, 2, 1, s))
torch.cuda.synchronize()
print("done")
