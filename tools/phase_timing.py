"""Per-phase CTA cycle breakdown of the block-solver kernel on the session's
hybrid layout (needs a build with EXTRA=-DTMG_PHASE_TIMING).  The figures are
those of the last launch of a sweep (the black colour's largest class).
usage: python tools/phase_timing.py [n]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08389_b200 import _lib, configs, grid, mgcycle  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
w = configs.workload("config3", n=n)
h = grid.build_hierarchy(w.x, w.x)
f = torch.from_numpy(w.rhs()).cuda()
u = torch.zeros_like(f)
L = _lib.lib()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
st = mgcycle._CycleState(h)
_lib.check(L.tmg_session_load(st.native, 4, ctypes.c_void_p(u.data_ptr()),
                              ctypes.c_void_p(f.data_ptr()), s))
out = (ctypes.c_double * 6)()
names = ["A gather", "B chunk elim", "reduced+PCR", "hub", "finalize", "C scatter"]
for rep in range(2):
    _lib.check(L.tmg_session_sweeps(st.native, 4, 1, s))
    torch.cuda.synchronize()
    nb = L.tmg_debug_phase_cycles(out)
tot = sum(out)
print(f"n={n} session sweep, last launch CTAs={nb} total={tot:.0f} cycles")
for k in range(6):
    print(f"   {names[k]:14s} {out[k]:9.0f}  {100 * out[k] / max(tot, 1):5.1f}%")
