"""V(2,2) cycle time of the config-3 recipe (tweed) at several sizes, on the
session graph: the differences between sizes give the per-level cost of the
coarse tail.  python tools/vcycle_sizes.py [n ...]"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08389_b200 import _lib, configs, grid, mgcycle  # noqa: E402

L = _lib.lib()
sizes = [int(a) for a in sys.argv[1:]] or [8, 16, 32, 64, 128, 256, 512, 1024, 2048]
for name in ("config3", "config1"):
    for n in sizes:
        w = configs.workload(name, n=n)
        h = grid.build_hierarchy(w.x, w.x)
        f = torch.from_numpy(w.rhs()).cuda()
        u = torch.zeros_like(f)
        st = mgcycle._CycleState(h)
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(L.tmg_session_load(st.native, 4, ctypes.c_void_p(u.data_ptr()),
                                      ctypes.c_void_p(f.data_ptr()), s))
        run = lambda r: _lib.check(L.tmg_session_cycles(st.native, 4, 1, 2, 2, r, s))  # noqa
        run(3)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        a.record()
        run(reps)
        b.record()
        torch.cuda.synchronize()
        print(json.dumps({"recipe": name, "n": n, "levels": len(h.levels),
                          "vcycle_ms": a.elapsed_time(b) / reps,
                          "kernels": int(L.tmg_last_kernels(st.native))
                          if hasattr(L, "tmg_last_kernels") else None}), flush=True)
        del st
