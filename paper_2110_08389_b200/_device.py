"""Device-buffer plumbing.  PyTorch supplies CUDA memory and streams only;
all arithmetic happens in the sm_100a library.

Operators accept CUDA float64 tensors (the native form) or numpy arrays
(the reference's form).  Numpy inputs are staged to the device, the GPU does
the work, and results come back as numpy, so reference-style callers keep
working unchanged.
"""

from __future__ import annotations

import ctypes

import numpy as np

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


def require_cuda():
    if torch is None or not torch.cuda.is_available():
        raise RuntimeError("paper_2110_08389_b200 needs a CUDA device (B200, sm_100a)")


def is_host(a) -> bool:
    return isinstance(a, np.ndarray)


def to_device(a, dtype=np.float64):
    """numpy -> contiguous CUDA tensor; CUDA tensors pass through (checked)."""
    require_cuda()
    dt = np.dtype(dtype)
    want = torch.float64 if dt == np.float64 else torch.int64
    if isinstance(a, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to("cuda")
    if not isinstance(a, torch.Tensor):
        raise TypeError(f"expected a numpy array or CUDA tensor, got {type(a).__name__}")
    if not a.is_cuda:
        a = a.to("cuda")
    if a.dtype != want:
        raise TypeError(f"expected {want} tensor, got {a.dtype}")
    if not a.is_contiguous():
        raise ValueError("tensor must be C-contiguous")
    return a


def shape_of(a):
    return tuple(a.shape)


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def stream_handle():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def empty(shape):
    return torch.empty(shape, dtype=torch.float64, device="cuda")


def zeros(shape):
    return torch.zeros(shape, dtype=torch.float64, device="cuda")


def back(t, like):
    """Return t in the caller's array flavour (numpy if `like` was numpy)."""
    if is_host(like):
        return t.cpu().numpy()
    return t
