"""A/B timing of one finest-level tweed sweep (both colours) and one V(2,2)
cycle of BASELINE config 3 on the loaded session: CUDA events around K
back-to-back sweeps (TMG_LEGK=0 selects the generic block kernel for every
block).  Prints one JSON line."""
import ctypes, json, os, sys
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
_lib.check(L.tmg_session_load(st.native, 4, ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(f.data_ptr()), s))


def ev(fn, reps):
    fn(1)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    fn(reps)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


sw = ev(lambda r: _lib.check(L.tmg_session_sweeps(st.native, 4, r, s)), 20)
cy = ev(lambda r: _lib.check(L.tmg_session_cycles(st.native, 4, 1, 2, 2, r, s)), 10)
n = w.x.n
alg = 24.0 * (n - 1) ** 2
print(json.dumps({"legk": os.environ.get("TMG_LEGK", "1"), "n": n, "sweep_ms": sw,
                  "sweep_GBs": alg / sw / 1e6, "frac": alg / sw / 1e6 / 6537.6,
                  "vcycle_ms": cy}))
