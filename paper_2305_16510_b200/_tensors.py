"""Planar (structure-of-arrays) fp32 device buffers and ctypes plumbing.

A batch of k-component records for n vehicles is one ``(k, stride)``
float32 CUDA tensor, ``stride = round_up(n, 4)``; component j of vehicle i
is ``buf[j, i]``.  API views keep the reference's shapes: e.g. positions are
``buf[0:3, :n].T`` with shape ``(n, 3)`` and strides ``(1, stride)``.
torch is used only for device memory and streams.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

DTYPE = torch.float32


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("a CUDA device is required (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def padded(n: int) -> int:
    return max(4, (int(n) + 3) // 4 * 4)


def alloc_planes(k: int, n: int, device=None, zero: bool = False) -> torch.Tensor:
    device = device if device is not None else default_device()
    fn = torch.zeros if zero else torch.empty
    return fn((k, padded(n)), dtype=DTYPE, device=device)


def as_device(x, device, dtype=DTYPE) -> torch.Tensor:
    """Array-like -> tensor on `device` (no copy when already there)."""
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype)
    return torch.as_tensor(np.asarray(x), dtype=dtype, device=device)


def pack_rows(buf: torch.Tensor, row0: int, x, n: int, width: int) -> None:
    """Copy an (n, width) (or (n,) when width == 1) array into planes."""
    t = as_device(x, buf.device)
    if width == 1:
        t = t.reshape(-1)
        if t.numel() == 1 and n != 1:
            t = t.expand(n)
        buf[row0, :n].copy_(t)
    else:
        t = t.reshape(-1, width)
        if t.shape[0] == 1 and n != 1:
            t = t.expand(n, width)
        buf[row0:row0 + width, :n].copy_(t.T)


def ptr(t) -> C.c_void_p:
    if t is None:
        return C.c_void_p(0)
    return C.c_void_p(t.data_ptr())


def stride0(t: torch.Tensor) -> int:
    return int(t.stride(0)) if t.dim() == 2 else int(t.numel())


def stream_handle(device=None) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)
