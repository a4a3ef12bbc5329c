"""Device-side argument handling shared by the drop-in API.

Arrays may be torch CUDA tensors (the fast path: no copies) or NumPy arrays
(the reference's own types): NumPy inputs are copied to the current CUDA
device, the kernel runs there, and results come back as NumPy arrays, so a
caller of the reference can swap the import and keep its code.  Nothing here
computes on the CPU.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from .errors import ConfigError

_SUFFIX = {torch.float32: "f32", torch.float64: "f64"}


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2511_17849_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(x, dtype: torch.dtype | None = None) -> tuple[torch.Tensor, bool]:
    """(flat contiguous CUDA tensor, came_from_numpy)."""
    if isinstance(x, np.ndarray):
        dev = require_cuda()
        src = torch.from_numpy(np.ascontiguousarray(x))
        t = src.to(dev, non_blocking=src.is_pinned())
        if dtype is not None and t.dtype != dtype:
            raise ConfigError(f"dtype mismatch: {t.dtype} vs {dtype}")
        return t.reshape(-1), True
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            raise ConfigError("tensor must live on a CUDA device (no CPU fallback)")
        if not x.is_contiguous():
            raise ConfigError("tensor must be contiguous")
        if dtype is not None and x.dtype != dtype:
            raise ConfigError(f"dtype mismatch: {x.dtype} vs {dtype}")
        return x.reshape(-1), False
    raise ConfigError(f"expected a torch CUDA tensor or a NumPy array, got {type(x).__name__}")


def suffix(t: torch.Tensor) -> str:
    try:
        return _SUFFIX[t.dtype]
    except KeyError:
        raise ConfigError(f"unsupported dtype {t.dtype}: float32 or float64") from None


def same_shape(*ts: torch.Tensor) -> int:
    n = ts[0].numel()
    for t in ts[1:]:
        if t.numel() != n or t.dtype != ts[0].dtype:
            raise ConfigError(
                f"participants disagree on shape/dtype: {tuple(t.shape)}/{t.dtype} vs "
                f"{tuple(ts[0].shape)}/{ts[0].dtype}")
    return n


def back(t: torch.Tensor, as_numpy: bool, shape=None):
    if not as_numpy:
        return t if shape is None else t.reshape(shape)
    a = t.cpu().numpy()
    return a if shape is None else a.reshape(shape)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def ptr_array(ts) -> C.Array:
    arr = (C.c_void_p * len(ts))()
    for i, t in enumerate(ts):
        arr[i] = t.data_ptr()
    return arr
