"""Bin-packing statistics of the block-solver plans (host only, no GPU).

python tools/plan_stats.py [n ...]   -> CTAs, slot fill and points per chunk
per colour for tweed (hybrid layout) and wireframe (hybrid layout).
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = ctypes.CDLL(os.path.join(ROOT, "paper_2110_08389_b200", "libtmg_b200.so"))

for n in [int(a) for a in sys.argv[1:]] or [1024, 8192]:
    for name, kind, mode in (("tweed", 4, 1), ("wireframe", 5, 2), ("zebra_x", 1, 3)):
        out = (ctypes.c_longlong * 8)()
        if L.tmg_plan_stats(kind, n, n, 16, mode, out) != 0:
            print(n, name, "failed")
            continue
        v = list(out)
        ctas, pts, thr = v[0] + v[4], v[2] + v[6], v[1] + v[5]
        print(f"{n:6d} {name:10s} CTAs {ctas:7d}  slot fill {pts / (ctas * 4096):.3f}  "
              f"thread fill {thr / (ctas * 256):.3f}  pts/chunk {pts / max(thr, 1):.2f}  "
              f"points {pts} / {(n - 1) ** 2}")
