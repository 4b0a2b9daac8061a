"""Phase cycles of the last sweep bin each tail CTA ran (library variant
built with -DTMG_PHASE_TIMING on tmg_sweep.cu):
TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_tailp.so python tools/tail_phases.py [n]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08389_b200 import _lib, configs, grid, mgcycle  # noqa: E402

L = _lib.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
w = configs.workload("config1", n=n)
h = grid.build_hierarchy(w.x, w.x)
f = torch.from_numpy(w.rhs()).cuda()
u = torch.zeros_like(f)
st = mgcycle._CycleState(h)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
_lib.check(L.tmg_session_load(st.native, 4, ctypes.c_void_p(u.data_ptr()),
                              ctypes.c_void_p(f.data_ptr()), s))
out = (ctypes.c_double * 6)()
_lib.check(L.tmg_session_cycles(st.native, 4, 1, 2, 2, 1, s))
torch.cuda.synchronize()
g4 = (ctypes.c_double * 4)()
L.tmg_debug_gather_cycles(g4)
nb = L.tmg_debug_phase_cycles(out)
names = ["A gather", "B chunk elim", "reduced+PCR", "hub", "finalize", "C scatter"]
print(f"n={n} ctas={nb} " + " ".join(f"{k}={v:.0f}" for k, v in zip(names, out)) +
      f" total={sum(out):.0f} cycles | gather: desc+wait={g4[0]:.0f} hub={g4[1]:.0f} "
      f"main={g4[2]:.0f} ends={g4[3]:.0f}")
