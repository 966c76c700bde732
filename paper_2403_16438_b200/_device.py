"""Tensor hand-off between numpy / torch and the C ABI (torch is plumbing only:
device memory, the current stream, and torch.distributed)."""
from __future__ import annotations

import numpy as np
import torch

from . import _lib

_DTYPES = {np.dtype(np.uint16): _lib.VB_U16, np.dtype(np.float32): _lib.VB_F32}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2403_16438_b200 needs a CUDA (sm_100a) device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def vb_dtype(t: torch.Tensor) -> int:
    if t.dtype == torch.uint16:
        return _lib.VB_U16
    if t.dtype == torch.float32:
        return _lib.VB_F32
    raise TypeError(f"unsupported frame dtype {t.dtype} (uint16 or float32)")


def as_device_frames(data, dev: torch.device | None = None) -> torch.Tensor:
    """(T,H,W) or (H,W) frames as a contiguous CUDA tensor of uint16 or float32.

    numpy uint16 stays uint16 (camera format, exact in float32); other numpy
    dtypes are widened to float32 like voltseg's Video (video_io.py:39-40)."""
    dev = dev or require_cuda()
    if isinstance(data, torch.Tensor):
        t = data
        if t.dtype not in (torch.uint16, torch.float32):
            t = t.to(torch.float32)
        return t.to(dev).contiguous()
    a = np.asarray(data)
    if a.dtype == np.uint16:
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).to(dev).view(torch.uint16)
    if a.dtype != np.float32:
        a = a.astype(np.float32)
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def empty_motion(n: int, dev: torch.device) -> torch.Tensor:
    return torch.empty(max(n, 1) * _lib.MOTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)


def motion_to_numpy(buf: torch.Tensor, n: int) -> np.ndarray:
    raw = buf[: n * _lib.MOTION_DTYPE.itemsize].cpu().numpy()
    return raw.view(_lib.MOTION_DTYPE).copy()


def ptr(t) -> int | None:
    """Device address of a tensor; raw integer addresses (IPC-mapped peer
    memory, which torch must not wrap -- it would copy it to the local device)
    pass through."""
    if t is None:
        return None
    return int(t) if isinstance(t, int) else t.data_ptr()
