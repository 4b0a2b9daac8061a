"""Subprocess worker for tests/test_gpu_tail.py: V-cycles of several smoother
kinds and sizes through the session graph (tmg_session_cycles), printing one
JSON line per case with a hash of the resulting u.  The test runs it with the
persistent coarse tail on (TMG_TAIL=1, tail_kernel in tmg_sweep.cu) and off
and requires identical hashes: the tail executes the same per-bin / per-tile
device code, so results are bit-identical."""

import ctypes
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2110_08389_b200 import _lib, configs, grid, mgcycle  # noqa: E402

CASES = [(4, "config1", 128), (4, "config3", 1024), (5, "config2", 128), (5, "config2", 512),
         (3, "config1", 256), (6, "config1", 128), (1, "config1", 64), (2, "config1", 64)]


def main():
    L = _lib.lib()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    for kind, name, n in CASES:
        w = configs.workload(name, n=n)
        h = grid.build_hierarchy(w.x, w.x)
        f = torch.from_numpy(w.rhs()).cuda()
        u = torch.zeros_like(f)
        st = mgcycle._CycleState(h)
        _lib.check(L.tmg_session_load(st.native, kind, P(u), P(f), s))
        for full, nu1, nu2 in ((1, 2, 1), (0, 1, 2), (1, 2, 2)):
            _lib.check(L.tmg_session_cycles(st.native, kind, full, nu1, nu2, 2, s))
        out = torch.empty_like(u)
        _lib.check(L.tmg_session_store(st.native, P(out), s))
        torch.cuda.synchronize()
        print(json.dumps({"kind": kind, "n": n, "recipe": name,
                          "hash": hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest(),
                          "finite": bool(torch.isfinite(out).all())}), flush=True)
        del st


if __name__ == "__main__":
    main()
