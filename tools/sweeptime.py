import ctypes, os, sys, time
sys.path.insert(0, "/root/repo") if os.path.exists("/root/repo") else None
sys.path.insert(0, os.getcwd())
import torch
from paper_2110_08389_b200 import _lib, configs, grid, mgcycle
from paper_2110_08389_b200.stencil import native_level
w = configs.workload("config3")
h = grid.build_hierarchy(w.x, w.x)
f = torch.from_numpy(w.rhs()).cuda(); u = torch.zeros_like(f)
L = _lib.lib(); st = mgcycle._CycleState(h)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
stream = torch.cuda.current_stream()
_lib.check(L.tmg_session_load(st.native, 4, ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(f.data_ptr()), s))
def ev(fn):
    torch.cuda.synchronize(); a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    t0=time.perf_counter(); a.record(stream); fn(); b.record(stream); t1=time.perf_counter(); torch.cuda.synchronize(); t2=time.perf_counter()
    return a.elapsed_time(b), (t1-t0)*1e3, (t2-t0)*1e3
for reps in (1,1,5,20):
    print("sweeps", reps, ev(lambda: _lib.check(L.tmg_session_sweeps(st.native, 4, reps, s))))
for reps in (1,1,5):
    print("cycles", reps, ev(lambda: _lib.check(L.tmg_session_cycles(st.native, 4, 1, 2, 2, reps, s))))
for reps in (1,5,20):
    print("sweeps", reps, ev(lambda: _lib.check(L.tmg_session_sweeps(st.native, 4, reps, s))))
lv = native_level(h.finest.stencil)
for reps in (1,5):
    print("api sweeps natural", reps, ev(lambda: [_lib.check(L.tmg_sweep(lv, 4, ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(f.data_ptr()), s)) for _ in range(reps)]))
