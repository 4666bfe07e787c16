"""Device plumbing: PyTorch is used only as the CUDA buffer / stream carrier."""

from __future__ import annotations

import numpy as np

from . import _lib

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda() -> None:
    """Fail loudly: the octree hot path has no CPU implementation."""
    _lib.load()
    if not torch().cuda.is_available():
        raise RuntimeError("the octree hot path needs a CUDA device (B200); none is visible")


def stream_handle() -> int:
    return torch().cuda.current_stream().cuda_stream


def ptr(t) -> int:
    return t.data_ptr()


def empty(shape, dtype_name: str):
    t = torch()
    return t.empty(shape, dtype=getattr(t, dtype_name), device="cuda")


def zeros(shape, dtype_name: str):
    t = torch()
    return t.zeros(shape, dtype=getattr(t, dtype_name), device="cuda")


def to_device_u8(frames):
    """A contiguous uint8 CUDA tensor view/copy of ``frames`` (numpy or torch)."""
    t = torch()
    if isinstance(frames, t.Tensor):
        if frames.dtype != t.uint8:
            raise ValueError(f"expected uint8 frames, got {frames.dtype}")
        x = frames if frames.is_cuda else frames.to("cuda", non_blocking=frames.is_pinned())
        return x.contiguous()
    arr = np.ascontiguousarray(frames)
    return t.from_numpy(arr).to("cuda")


def frames_on_device(frames, what: str = "frames"):
    """Validated (n, h, w, 3) uint8 frames as a contiguous CUDA tensor on the
    current device, for the batched device entry points: a strided view is
    made contiguous, host data (numpy / CPU tensor) is copied over, and a
    tensor on another CUDA device is rejected -- the kernels take a raw
    pointer and would otherwise read wrong pixels or fault."""
    t = torch()
    if isinstance(frames, t.Tensor):
        shape, ok_dtype = tuple(frames.shape), frames.dtype == t.uint8
        if frames.is_cuda and frames.device.index != t.cuda.current_device():
            raise ValueError(f"{what} are on {frames.device}, the current device is cuda:{t.cuda.current_device()}")
    else:
        frames = np.asarray(frames)
        shape, ok_dtype = frames.shape, frames.dtype == np.uint8
    if len(shape) != 4 or shape[3] != 3 or not ok_dtype:
        raise ValueError(f"{what}: expected (n, h, w, 3) uint8 frames, got {frames.dtype} {shape}")
    return to_device_u8(frames)


def to_device_u32(arr):
    t = torch()
    if isinstance(arr, t.Tensor):
        return arr.to("cuda").contiguous()
    a = np.ascontiguousarray(arr, dtype=np.uint32)
    return t.from_numpy(a.view(np.int32)).to("cuda")


def u32_to_numpy(tensor) -> np.ndarray:
    """Device int32-typed words -> host uint32 ndarray."""
    return tensor.detach().cpu().numpy().view(np.uint32)


def is_tensor(x) -> bool:
    try:
        return isinstance(x, torch().Tensor)
    except ImportError:  # pragma: no cover
        return False


# ---------------------------------------------------------------------------
# Host staging for the reference-signature path (numpy frames in, numpy masks
# out): frames are gathered into pinned buffers by libobg's persistent host
# copy pool (obg_host_gather, GIL released) and moved with asynchronous H2D
# copies -- instead of np.stack (one single-threaded 400 MB copy for 64 C3
# frames) followed by a pageable H2D.  Buffers are cached per thread.
# ---------------------------------------------------------------------------
import ctypes
import threading

_TLS = threading.local()
_STAGE_BYTES = 64 << 20                 # frames per staging chunk: ~64 MiB


def _pinned(key, shape):
    """Thread-local pinned uint8 buffer + the event of its last async use."""
    cache = getattr(_TLS, "pinned", None)
    if cache is None:
        cache = _TLS.pinned = {}
    ent = cache.get(key)
    if ent is None or tuple(ent[0].shape) != tuple(shape):
        t = torch()
        ent = [t.empty(shape, dtype=t.uint8, pin_memory=True), None]
        cache[key] = ent
    return ent


def host_gather(arrays, dst_ptr: int, nbytes: int) -> None:
    """Copy equally sized contiguous host arrays back to back into dst_ptr."""
    srcs = (ctypes.c_void_p * len(arrays))(*[a.ctypes.data for a in arrays])
    _lib.check(_lib.load().obg_host_gather(srcs, len(arrays), nbytes, dst_ptr))


def frames_list_to_device(frames):
    """A list of (h, w, 3) uint8 numpy frames as one (n, h, w, 3) CUDA tensor
    on the current device / stream: chunks gathered into two alternating
    pinned buffers while the previous chunk's H2D runs."""
    t = torch()
    n = len(frames)
    h, w = frames[0].shape[:2]
    fb = h * w * 3
    dev = t.empty((n, h, w, 3), dtype=t.uint8, device="cuda")
    k = max(1, min(n, _STAGE_BYTES // max(fb, 1)))
    stream = t.cuda.current_stream()
    for c, s0 in enumerate(range(0, n, k)):
        m = min(k, n - s0)
        ent = _pinned(("stage", c & 1, h, w), (k, h, w, 3))
        if ent[1] is not None:
            ent[1].synchronize()                     # the slot's previous H2D has read it
        chunk = [np.ascontiguousarray(f) for f in frames[s0:s0 + m]]
        host_gather(chunk, ent[0].data_ptr(), fb)
        dev[s0:s0 + m].copy_(ent[0][:m], non_blocking=True)
        ev = t.cuda.Event()
        ev.record(stream)
        ent[1] = ev
    return dev
