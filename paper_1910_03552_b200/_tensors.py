"""Small host helpers: numpy/torch in, contiguous CUDA tensors out."""
from __future__ import annotations

import contextlib
import gc

import numpy as np
import torch

from ._native import require_cuda
from .errors import SchemaError

_status_words: dict[int, "object"] = {}


@contextlib.contextmanager
def graph_capture(graph, **kw):
    """`torch.cuda.graph(graph, **kw)` with Python's cyclic garbage collector paused.

    torch no longer collects garbage when a capture begins. An automatic collection that runs
    mid-capture can finalise an unreachable CUDAGraph from earlier work, and destroying its
    executable is an unsafe call that invalidates a global-mode capture. Seen as "operation
    failed due to a previous error during capture" at the next launch."""
    enabled = gc.isenabled()
    gc.disable()
    try:
        with torch.cuda.graph(graph, **kw):
            yield
    finally:
        if enabled:
            gc.enable()


def status_word(device: torch.device):
    from .errors import StatusWord

    idx = device.index if device.index is not None else torch.cuda.current_device()
    sw = _status_words.get(idx)
    if sw is None:
        sw = StatusWord(device=torch.device("cuda", idx))
        _status_words[idx] = sw
    return sw


def to_cuda(x, dtype: torch.dtype, device=None) -> tuple[torch.Tensor, bool]:
    """Return (contiguous CUDA tensor of `dtype`, input_was_numpy)."""
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            require_cuda()
            x = x.to(device or "cuda")
        if x.dtype != dtype:
            x = x.to(dtype)
        return x.contiguous(), False
    arr = np.asarray(x)
    require_cuda()
    t = torch.from_numpy(np.ascontiguousarray(arr)).to(device or "cuda")
    if t.dtype != dtype:
        t = t.to(dtype)
    return t, True


def out_like(t: torch.Tensor, as_numpy: bool, np_dtype=np.float32):
    if not as_numpy:
        return t
    return t.detach().cpu().numpy().astype(np_dtype, copy=False)


def expect_shape(name: str, t, shape: tuple) -> None:
    if tuple(t.shape) != tuple(shape):
        raise SchemaError(f"{name} shape {tuple(t.shape)}, expected {tuple(shape)}")
