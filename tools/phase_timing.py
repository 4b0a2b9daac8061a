"""Per-phase CTA cycle breakdown of the block-solver kernel (needs a build
with EXTRA=-DTMG_PHASE_TIMING).  usage: python tools/phase_timing.py [n]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08389_b200 import _lib, configs, grid  # noqa: E402
from paper_2110_08389_b200.stencil import native_level  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
w = configs.workload("config3", n=n)
st = grid.Level(w.x, w.x).stencil
f = torch.from_numpy(w.rhs()).cuda()
u = torch.zeros_like(f)
L = _lib.lib()
L.tmg_debug_phase_cycles.argtypes = [ctypes.POINTER(ctypes.c_double)]
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
lv = native_level(st)
out = (ctypes.c_double * 6)()
names = ["A gather", "B chunk elim", "reduced+PCR", "hub", "finalize", "C scatter"]
for colour in (1, 0):
    for rep in range(2):
        _lib.check(L.tmg_sweep_colour(lv, 4, colour, ctypes.c_void_p(u.data_ptr()),
                                      ctypes.c_void_p(f.data_ptr()), s))
        torch.cuda.synchronize()
        nb = L.tmg_debug_phase_cycles(out)
    tot = sum(out)
    print(f"n={n} colour={'red' if colour else 'black'} CTAs={nb} total={tot:.0f} cycles")
    for k in range(6):
        print(f"   {names[k]:14s} {out[k]:9.0f}  {100 * out[k] / max(tot, 1):5.1f}%")
