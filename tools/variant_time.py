"""Time finest-level sweeps and V-cycles of config 3 on the session layout
(A/B runs of library variants: run once per variant .so in its own process).
python tools/variant_time.py [--n N] [--kind tweed]"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08389_b200 import _lib, configs, grid, mgcycle  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=None)
p.add_argument("--kind", default="tweed")
p.add_argument("--tag", default="")
a = p.parse_args()
w = configs.workload("config3", n=a.n)
h = grid.build_hierarchy(w.x, w.x)
f = torch.from_numpy(w.rhs()).cuda()
u = torch.zeros_like(f)
L = _lib.lib()
st = mgcycle._CycleState(h)
k = _lib.KIND_IDS[a.kind]
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
stream = torch.cuda.current_stream()
_lib.check(L.tmg_session_load(st.native, k, ctypes.c_void_p(u.data_ptr()),
                              ctypes.c_void_p(f.data_ptr()), s))


def ev(fn, reps):
    fn(2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fn(reps)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


sw = ev(lambda r: _lib.check(L.tmg_session_sweeps(st.native, k, r, s)), 20)
cy = ev(lambda r: _lib.check(L.tmg_session_cycles(st.native, k, 1, 2, 2, r, s)), 10)
print(f"{a.tag:10s} sweep {sw:.4f} ms  V(2,2) {cy:.4f} ms")
