"""Device plumbing: tensors, streams, workspaces, host<->device transfers.

PyTorch is used only as the allocator / stream provider; all compute goes
through the C ABI.  Host outputs are staged in pinned memory (torch's caching
host allocator) and handed back as numpy views, so D2H runs at full PCIe
speed and no extra host copy is made.
"""

from __future__ import annotations

import warnings

import numpy as np
import torch

from . import _lib

_NP2T = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
         np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64,
         np.dtype(np.uint8): torch.uint8, np.dtype(np.uint32): torch.uint32}


_DEVICES = {}  # current device index -> torch.device (the library checked once)


def device() -> torch.device:
    if not _DEVICES:
        _lib.lib()  # asserts CUDA + library (the reference's errors without them)
    idx = torch.cuda.current_device()
    d = _DEVICES.get(idx)
    if d is None:
        d = _DEVICES[idx] = torch.device("cuda", idx)
    return d


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream() -> int:
    """cudaStream_t of torch's current stream (the raw getter skips building a
    Stream object: this is on every call's host path)."""
    if _RAW_STREAM is not None:
        return _RAW_STREAM(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def empty(shape, dtype, dev=None) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=dev or device())


def workspace(nbytes: int) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device())


def is_cuda_tensor(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def h2d(arr: np.ndarray) -> torch.Tensor:
    """Host numpy -> device tensor (async from pinned memory, else staged)."""
    arr = np.ascontiguousarray(arr)
    if not arr.flags.writeable:  # torch warns on read-only views; we never write them
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)
            t = torch.from_numpy(arr)
    else:
        t = torch.from_numpy(arr)
    return t.to(device(), non_blocking=True)


def as_tensor(arr: np.ndarray) -> torch.Tensor:
    """Zero-copy host tensor view of a numpy array (read-only views allowed)."""
    arr = np.ascontiguousarray(arr)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(arr)


def is_pinned(arr: np.ndarray) -> bool:
    """True when the array's memory is page-locked (cudaHostAlloc'ed)."""
    try:
        return bool(as_tensor(arr).is_pinned())
    except Exception:
        return False


def pinned(shape, dtype) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, pin_memory=True)


def d2h(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> numpy view of a pinned host buffer (sync)."""
    host = pinned(tuple(t.shape), t.dtype)
    host.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return host.numpy()


def d2h_many(*ts) -> list:
    hosts = []
    for t in ts:
        if t is None:
            hosts.append(None)
            continue
        h = pinned(tuple(t.shape), t.dtype)
        h.copy_(t, non_blocking=True)
        hosts.append(h)
    torch.cuda.current_stream().synchronize()
    return [None if h is None else h.numpy() for h in hosts]


class Status:
    """A device status word plus a pinned readback slot."""

    def __init__(self):
        self.dev = torch.zeros(1, dtype=torch.int32, device=device())

    @property
    def ptr(self) -> int:
        return self.dev.data_ptr()

    def read(self) -> int:
        return int(d2h(self.dev)[0]) & 0xFFFFFFFF
