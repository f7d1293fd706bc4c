"""Device marshalling for the operator-level entry points (numpy-in/numpy-out like the
reference, or CUDA tensors in and out).  Every apply runs in libbbdg_cuda.so; there is no
host fallback."""

from __future__ import annotations

import numpy as np

from . import _lib


def torch():
    import torch as _t  # plumbing only: device buffers and streams

    if not _t.cuda.is_available():
        raise _lib.BBDGError("no CUDA device: the BB-DG operators run only on the GPU (no CPU fallback)")
    return _t


def is_tensor(x) -> bool:
    return type(x).__module__.startswith("torch")


def to_device(x, dtype=None):
    """(contiguous CUDA tensor, was_host) for a numpy array or tensor; float32/float64 kept
    (other dtypes become float64, as numpy promotes in the reference)."""
    t = torch()
    host = not is_tensor(x)
    if host:
        a = np.asarray(x)
        if dtype is None:
            dtype = a.dtype if a.dtype in (np.float32, np.float64) else np.float64
        d = t.from_numpy(np.ascontiguousarray(a, dtype=dtype)).cuda()
    else:
        d = x if x.is_cuda else x.cuda()
        if d.dtype not in (t.float32, t.float64):
            d = d.to(t.float64)
        d = d.contiguous()
    return d, host


def back(d, host):
    return d.cpu().numpy() if host else d


def dtype_id(d) -> int:
    return 0 if d.dtype == torch().float32 else 1


def stream() -> int:
    return torch().cuda.current_stream().cuda_stream


_tables: dict = {}


def table(key, array: np.ndarray, like):
    """Device copy of a host float64 table in the dtype of `like` (cached per device/dtype)."""
    t = torch()
    k = (key, like.dtype, like.device)
    d = _tables.get(k)
    if d is None:
        d = t.as_tensor(np.ascontiguousarray(array, dtype=np.float64), device=like.device).to(like.dtype)
        _tables[k] = d
    return d


def dense_apply(key, A: np.ndarray, x, nrows: int | None = None):
    """y = x A^T on the device (opcount.dense_apply, reference opcount.py:38-43)."""
    A = np.asarray(A)
    xd, host = to_device(x)
    if xd.shape[-1] != A.shape[1]:
        raise ValueError(f"expected trailing size {A.shape[1]}, got {xd.shape[-1]}")
    Ad = table(key, A, xd)
    y = torch().empty(tuple(xd.shape[:-1]) + (A.shape[0],), dtype=xd.dtype, device=xd.device)
    nb = xd.numel() // A.shape[1] if A.shape[1] else 0
    _lib.check(_lib.load().bbdg_dense_apply(dtype_id(xd), nb, A.shape[0], A.shape[1], Ad.data_ptr(), xd.data_ptr(),
                                            y.data_ptr(), stream()), "bbdg_dense_apply")
    return back(y, host)
