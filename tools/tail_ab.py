"""Cycle results with and without the persistent coarse tail: runs a few
V-cycles per (kind, size) and prints a hash of u and the cycle time; run it
once with TMG_TAIL=0 and once without to compare bit for bit."""
import ctypes
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2110_08389_b200 import _lib, configs, grid, mgcycle  # noqa: E402

L = _lib.lib()
cases = [(4, "config1", 128), (4, "config3", 64), (4, "config3", 1024), (5, "config2", 128),
         (5, "config2", 1024), (3, "config1", 256), (6, "config1", 256), (1, "config1", 64),
         (0, "config1", 64)]
for kind, name, n in cases:
    w = configs.workload(name, n=n)
    h = grid.build_hierarchy(w.x, w.x)
    f = torch.from_numpy(w.rhs()).cuda()
    u = torch.zeros_like(f)
    st = mgcycle._CycleState(h)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(L.tmg_session_load(st.native, kind, ctypes.c_void_p(u.data_ptr()),
                                  ctypes.c_void_p(f.data_ptr()), s))
    for full in (1, 0):
        _lib.check(L.tmg_session_cycles(st.native, kind, full, 2, 1, 3, s))
    out = torch.empty_like(u)
    _lib.check(L.tmg_session_store(st.native, ctypes.c_void_p(out.data_ptr()), s))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check(L.tmg_session_cycles(st.native, kind, 1, 2, 2, 20, s))
    b.record()
    torch.cuda.synchronize()
    hsh = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps({"kind": kind, "recipe": name, "n": n, "hash": hsh,
                      "absmax": float(out.abs().max()), "vcycle_ms": a.elapsed_time(b) / 20}),
          flush=True)
    del st
