"""Device plumbing: PyTorch owns device memory and streams; the CUDA library
only ever sees raw pointers (see include/cspq_b200.h)."""

from __future__ import annotations

import numpy as np

from ._native import require_cuda


def torch():
    import torch as _t
    return _t


def device(index: int | None = None):
    require_cuda()
    t = torch()
    return t.device("cuda", t.cuda.current_device() if index is None else index)


def stream_ptr(dev=None) -> int:
    t = torch()
    return t.cuda.current_stream(dev).cuda_stream


def ptr(x) -> int | None:
    if x is None:
        return None
    return x.data_ptr()


def to_device(a, dev, dtype=None):
    """numpy/torch -> contiguous CUDA tensor on dev (async from pinned memory)."""
    t = torch()
    if isinstance(a, t.Tensor):
        x = a
    else:
        a = np.ascontiguousarray(a)
        x = t.from_numpy(a if a.flags.writeable else a.copy())
    if dtype is not None and x.dtype != dtype:
        x = x.to(dtype)
    return x.to(dev, non_blocking=True).contiguous()


def pinned_empty(shape, dtype=np.float32) -> np.ndarray:
    """A numpy array backed by page-locked host memory (cudaHostAlloc through
    torch), so host<->device copies run at PCIe speed and asynchronously."""
    t = torch()
    tdt = {np.dtype(np.float32): t.float32, np.dtype(np.uint8): t.uint8,
           np.dtype(np.uint16): t.int16, np.dtype(np.int32): t.int32,
           np.dtype(np.float64): t.float64}[np.dtype(dtype)]
    buf = t.empty(tuple(shape), dtype=tdt, pin_memory=True)
    arr = buf.numpy()
    if np.dtype(dtype) == np.uint16:
        arr = arr.view(np.uint16)
    _KEEP[id(arr)] = buf  # keep the pinned allocation alive with the array
    return arr


_KEEP: dict = {}
