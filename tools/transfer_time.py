"""Time the finest-level residual+restriction, prolongation+correction and
residual norm of config 3 on the session layout (CUDA events), with the
algorithmic bandwidth of each.  python tools/transfer_time.py [--tag T]"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08389_b200 import _lib, configs, grid, mgcycle  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--tag", default="")
p.add_argument("--n", type=int, default=None)
a = p.parse_args()
w = configs.workload("config3", n=a.n)
h = grid.build_hierarchy(w.x, w.x)
f = torch.from_numpy(w.rhs()).cuda()
u = torch.zeros_like(f)
L = _lib.lib()
st = mgcycle._CycleState(h)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
stream = torch.cuda.current_stream()
_lib.check(L.tmg_session_load(st.native, 4, ctypes.c_void_p(u.data_ptr()),
                              ctypes.c_void_p(f.data_ptr()), s))
_lib.check(L.tmg_session_sweeps(st.native, 4, 1, s))


def ev(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


nf = (h.finest.nx + 1) * (h.finest.ny + 1)
nc = (h.levels[1].nx + 1) * (h.levels[1].ny + 1)
tr = ev(lambda: _lib.check(L.tmg_session_restrict(st.native, 0, 1, s)))
tp = ev(lambda: _lib.check(L.tmg_session_prolong(st.native, 0, s)))
out = ctypes.c_double()
tn = ev(lambda: _lib.check(L.tmg_session_norm(st.native, ctypes.byref(out), s)), 5)
for name, t, b in (("restrict", tr, 16 * nf + 8 * nc), ("prolong", tp, 16 * nf + 8 * nc),
                   ("norm(+sync)", tn, 16 * nf)):
    print(f"{a.tag:6s} {name:12s} {t * 1e3:8.1f} us  {b / t / 1e6:7.0f} GB/s")
print(f"{a.tag:6s} norm value {out.value!r}")
