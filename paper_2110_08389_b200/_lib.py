"""ctypes binding of the native library (include/tweedmg_b200.h).

The CUDA library is the only compute path: if it is missing or cannot be
loaded, every operator raises instead of falling back to CPU code.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TMG_LIB_PATH") or os.path.join(_HERE, "libtmg_b200.so")  # override: A/B runs

TMG_OK, TMG_SINGULAR, TMG_BADARG, TMG_CUDA = 0, 1, 2, 3

KIND_IDS = {
    "checkerboard": 0, "zebra_x": 1, "zebra_y": 2, "zebra_alt": 3,
    "tweed": 4, "wireframe": 5, "tweed_wire_alt": 6,
}

_lib = None
_load_error = None


class NativeLibraryError(RuntimeError):
    """The sm_100a library is not built or cannot be loaded."""


def _declare(L):
    vp, ip, dp = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
    lp = ctypes.c_long
    pi = ctypes.POINTER(ctypes.c_int)
    pd = ctypes.POINTER(ctypes.c_double)
    sig = {
        "tmg_last_error": ([], ctypes.c_char_p),
        "tmg_version": ([], ip),
        "tmg_level_create": ([ip, ip, vp, vp, vp, vp, ctypes.POINTER(vp)], ip),
        "tmg_level_destroy": ([vp], ip),
        "tmg_level_device_bytes": ([vp], ctypes.c_longlong),
        "tmg_level_check": ([vp, vp], ip),
        "tmg_sweep": ([vp, ip, vp, vp, vp], ip),
        "tmg_sweep_colour": ([vp, ip, ip, vp, vp, vp], ip),
        "tmg_apply": ([vp, vp, vp, vp], ip),
        "tmg_defect": ([vp, vp, vp, vp, vp], ip),
        "tmg_defect_norm": ([vp, vp, vp, pd, vp], ip),
        "tmg_restrict": ([ip, ip, ip, vp, vp, vp], ip),
        "tmg_prolong": ([ip, ip, vp, vp, vp], ip),
        "tmg_defect_restrict": ([vp, ip, vp, vp, vp, vp], ip),
        "tmg_prolong_correct": ([ip, ip, vp, vp, vp], ip),
        "tmg_direct_solve": ([vp, vp, vp, vp], ip),
        "tmg_hier_create": ([ip, ctypes.POINTER(vp), ctypes.POINTER(vp)], ip),
        "tmg_hier_destroy": ([vp], ip),
        "tmg_vcycle": ([vp, ip, ip, ip, ip, vp, vp, vp], ip),
        "tmg_vcycle_graph": ([vp, ip, ip, ip, ip, vp, vp, ip, vp], ip),
        "tmg_hier_graph_kernels": ([vp], ip),
        "tmg_hier_device_bytes": ([vp], ctypes.c_longlong),
        "tmg_session_load": ([vp, ip, vp, vp, vp], ip),
        "tmg_session_cycles": ([vp, ip, ip, ip, ip, ip, vp], ip),
        "tmg_session_norm": ([vp, pd, vp], ip),
        "tmg_session_store": ([vp, vp, vp], ip),
        "tmg_session_sweeps": ([vp, ip, ip, vp], ip),
        "tmg_debug_phase_cycles": ([pd], ip),
        "tmg_kernel_launches": ([], ctypes.c_longlong),
        "tmg_vec_norm2": ([vp, lp, vp, pd, vp], ip),
        "tmg_vec_scale": ([vp, lp, dp, vp], ip),
        "tmg_lcg_fill": ([ctypes.c_ulonglong, lp, vp, vp], ip),
        "tmg_cube_last_error": ([], ctypes.c_char_p),
        "tmg_cube_create": ([ip, vp, ctypes.POINTER(vp)], ip),
        "tmg_cube_create_scheme": ([ip, vp, ip, ctypes.POINTER(vp)], ip),
        "tmg_cube_destroy": ([vp], ip),
        "tmg_cube_levels": ([vp], ip),
        "tmg_cube_blocks": ([vp, ip, ip], lp),
        "tmg_cube_sweep": ([vp, vp, vp, vp], ip),
        "tmg_cube_defect": ([vp, vp, vp, vp, vp], ip),
        "tmg_cube_load": ([vp, vp, vp, vp], ip),
        "tmg_cube_cycles": ([vp, ip, ip, ip, vp], ip),
        "tmg_cube_norm": ([vp, pd, vp], ip),
        "tmg_cube_solve_loop": ([vp, ip, ip, dp, dp, ip, pd, pi, pi, vp], ip),
        "tmg_cube_store": ([vp, vp, vp], ip),
        "tmg_cube_sweeps": ([vp, ip, vp], ip),
        "tmg_cube_group_count": ([ip, ip], ip),
        "tmg_cube_group_sizes": ([ip, ip, vp, lp], lp),
        "tmg_cube_group_offsets": ([ip, ip, ip, ip, vp, lp], lp),
        "tmg_cube_sweep_part": ([vp, ip, ip, ip, ip, vp], ip),
        "tmg_cube_restrict": ([vp, ip, vp], ip),
        "tmg_cube_prolong": ([vp, ip, vp], ip),
        "tmg_cube_tail": ([vp, ip, ip, ip, vp], ip),
        "tmg_cube_gather": ([vp, ip, ip, vp, lp, vp, vp], ip),
        "tmg_cube_scatter": ([vp, ip, ip, vp, lp, vp, vp], ip),
        "tmg_cube_norm_part": ([vp, ip, ip, pd, vp], ip),
        "tmg_group_count": ([ip, ip, ip], ip),
        "tmg_group_sizes": ([ip, ip, ip, vp, lp], lp),
        "tmg_group_offsets": ([ip, ip, ip, ip, ip, vp, lp], lp),
        "tmg_session_sweep_part": ([vp, ip, ip, ip, ip, ip, vp], ip),
        "tmg_session_restrict": ([vp, ip, ip, vp], ip),
        "tmg_session_read": ([vp, ip, ip, vp, vp], ip),
        "tmg_session_restrict_part": ([vp, ip, ip, ip, ip, ip, vp], ip),
        "tmg_session_prolong_part": ([vp, ip, ip, ip, ip, vp], ip),
        "tmg_session_prolong": ([vp, ip, vp], ip),
        "tmg_session_tail": ([vp, ip, ip, ip, ip, ip, vp], ip),
        "tmg_session_gather": ([vp, ip, ip, vp, lp, vp, vp], ip),
        "tmg_session_scatter": ([vp, ip, ip, vp, lp, vp, vp], ip),
        "tmg_session_norm_part": ([vp, ip, ip, ip, pd, vp], ip),
        "tmg_session_check": ([vp, vp], ip),
        "tmg_solve": ([vp, ip, ip, ip, ip, dp, ip, vp, vp, pd, pi, pi, vp], ip),
        "tmg_layout_dump": ([ip, ip, ip, pi, pi, pi, pi, lp], lp),
        "tmg_relax_points": ([lp, vp, vp, ip, ip, vp, vp, vp, vp, vp, vp, vp], ip),
        "tmg_relax_chain": ([lp, vp, vp, ip, ip, vp, vp, vp, vp, vp, vp, vp], ip),
        "tmg_relax_ring": ([lp, vp, vp, ip, ip, vp, vp, vp, vp, vp, vp, vp], ip),
        "tmg_relax_legged": ([lp, vp, vp, lp, vp, lp, lp, ip, ip, vp, vp, vp, vp, vp, vp, vp], ip),
        "tmg_thomas": ([lp, vp, vp, vp, vp, vp, vp], ip),
        "tmg_circulant_thomas": ([lp, vp, vp, vp, vp, vp, vp], ip),
        "tmg_legged_thomas": ([lp, vp, vp, vp, vp, vp, vp, dp, dp, vp, vp, vp], ip),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return sig


def lib():
    """Load (once) and return the native library; raises if unavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"native library {LIB_PATH} is not built; run __graft_entry__.build()")
    try:
        L = ctypes.CDLL(LIB_PATH)
        _declare(L)
    except OSError as exc:  # pragma: no cover - depends on the box
        _load_error = exc
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
    _lib = L
    return L


def exported_symbols():
    """Names declared by include/tweedmg_b200.h that the loader binds."""
    L = lib()
    return sorted(n for n in _declare(L))


def available() -> bool:
    try:
        lib()
        return True
    except NativeLibraryError:
        return False


def check(status: int):
    """Map a C-ABI status to the reference's exception types."""
    if status == TMG_OK:
        return
    msg = lib().tmg_last_error().decode(errors="replace")
    if status == TMG_SINGULAR:
        from .tridiag import SingularSystemError
        raise SingularSystemError(msg)
    if status == TMG_BADARG:
        raise ValueError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


def host_ptr(a: np.ndarray):
    assert a.flags.c_contiguous
    return ctypes.c_void_p(a.ctypes.data)
