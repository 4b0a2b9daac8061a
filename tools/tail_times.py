"""Per-op timeline of the persistent coarse tail (CTA 0, %globaltimer):
work = op start -> op end, wait = op end -> next op start (the barrier).
Needs the TMG_TAIL_TIMING library variant:
TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_tailt.so python tools/tail_times.py [n]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
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
_lib.check(L.tmg_session_cycles(st.native, 4, 1, 2, 2, 3, s))
torch.cuda.synchronize()
buf = np.zeros(2 * 4096, dtype=np.uint64)
L.tmg_debug_tail_times(ctypes.c_void_p(buf.ctypes.data), 4096)
t0, t1 = buf[:4096].astype(np.int64), buf[4096:].astype(np.int64)
k = int(np.argmax(t0 == 0)) if (t0 == 0).any() else 4096
print(f"n={n} ops={k} total={(t1[k - 1] - t0[0]) / 1e3:.1f} us")
for i in range(k):
    wait = (t0[i + 1] - t1[i]) / 1e3 if i + 1 < k else 0.0
    print(f"op {i:3d} work {(t1[i] - t0[i]) / 1e3:7.2f} us  wait {wait:7.2f} us")
