"""Golden fixtures of the reference's per-colour index plans
(tweedmg.smoothers.compile_plan, smoothers.py:92-104) -> plans.npz.

Run in the build container, where the reference is importable:
    python tests/golden/make_plans_golden.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref", "src"))
sys.path.insert(0, HERE)

from tweedmg import smoothers  # noqa: E402

from plan_codec import SCHEMES, SIZES, flatten_plans  # noqa: E402


def main():
    out = {}
    for scheme in SCHEMES:
        for nx, ny in SIZES:
            out.update(flatten_plans(f"{scheme}_{nx}x{ny}", smoothers.compile_plan(scheme, nx, ny)))
    np.savez_compressed(os.path.join(HERE, "plans.npz"), **out)
    print(len(out), "arrays")


if __name__ == "__main__":
    main()
