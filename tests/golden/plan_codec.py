"""Flat encoding of {"red": ColourPlan, "black": ColourPlan} (the reference's
smoothers.py:25-34 plan objects) as named int64 arrays, shared by the golden
generator and tests/test_plans.py."""

import numpy as np

SCHEMES = ("checkerboard", "zebra_x", "zebra_y", "tweed", "wireframe")
SIZES = ((8, 8), (12, 10), (10, 14), (20, 8), (6, 16))


def _cat(parts):
    return np.concatenate(parts).astype(np.int64) if parts else np.empty(0, np.int64)


def flatten_plans(tag, plans):
    out = {}
    for colour in ("red", "black"):
        p = plans[colour]
        t = f"{tag}_{colour}"
        out[f"{t}_points"] = np.stack([np.asarray(p.points_i, np.int64),
                                       np.asarray(p.points_j, np.int64)])
        out[f"{t}_leg_ii"] = _cat([np.asarray(b[0]) for b in p.legged])
        out[f"{t}_leg_jj"] = _cat([np.asarray(b[1]) for b in p.legged])
        out[f"{t}_leg_offs"] = _cat([np.asarray(b[2]) for b in p.legged])
        out[f"{t}_leg_hub"] = np.array([[b[3], b[4]] for b in p.legged], np.int64).reshape(-1, 2)
        out[f"{t}_leg_n"] = np.array([len(b[0]) for b in p.legged], np.int64)
        for key, lst in (("chain", p.chains), ("ring", p.rings)):
            out[f"{t}_{key}_ii"] = _cat([np.asarray(b[0]) for b in lst])
            out[f"{t}_{key}_jj"] = _cat([np.asarray(b[1]) for b in lst])
            out[f"{t}_{key}_n"] = np.array([len(b[0]) for b in lst], np.int64)
    return out
