"""Per-pixel foreground classification (reference detect.py:22-53) on the GPU.

``detect_octree`` keeps the reference's single-frame signature (numpy in,
``(h, w)`` bool out).  ``classify`` is the batched device entry point: many
frames per launch, masks written straight into a device buffer, optionally
bit-packed.
"""

from __future__ import annotations

import numpy as np

from . import _device, _lib
from .model import BackgroundModel


def _check_frame_shape(model: BackgroundModel, h: int, w: int) -> None:
    if (h, w) != (model.frame_height, model.frame_width):
        raise ValueError(f"frame is {w}x{h}, model expects {model.frame_width}x{model.frame_height}")


def classify(model: BackgroundModel, frames_dev, out=None, packed: bool = False, after_build: bool = False):
    """Foreground masks of a (n, h, w, 3) uint8 CUDA tensor.

    ``after_build``: the previous work on the current stream is the
    ``build_background_model_device`` call that produced ``model`` (the
    captured step): the kernel is launched as a programmatic dependent of the
    merge kernel (``OBG_MASK_AFTER_MODEL``), removing the launch gap.

    Returns (and fills ``out`` if given) a uint8 CUDA tensor: ``(n, h, w)``
    0/1 bytes, or ``(n, ceil(h*w/8))`` LSB-first bits when ``packed``.
    A pixel is foreground iff its quantized colour is not a full-depth leaf
    of its region's merged tree; an empty tree flags everything (detect.py:44-52).
    """
    frames_dev = _device.frames_on_device(frames_dev)
    n, h, w = int(frames_dev.shape[0]), int(frames_dev.shape[1]), int(frames_dev.shape[2])
    _check_frame_shape(model, h, w)
    cfg = model.config
    cube = model.device_cube()
    shape = (n, (h * w + 7) // 8) if packed else (n, h, w)
    if out is None:
        out = _device.empty(shape, "uint8")
    elif tuple(out.shape) != shape or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous {shape} uint8 tensor")
    lib = _lib.load()
    _lib.check(lib.obg_classify(_device.ptr(frames_dev), n, h, w, cfg.levels, cfg.grid_rows, cfg.grid_cols,
                                _device.ptr(cube), _device.ptr(out),
                                (_lib.MASK_PACKED if packed else _lib.MASK_U8) |
                                (_lib.MASK_AFTER_MODEL if after_build else 0), _device.stream_handle()))
    return out


def _detect_host(model: BackgroundModel, frames: np.ndarray) -> np.ndarray:
    """(n, h, w, 3) uint8 numpy frames -> (n, h, w) bool numpy masks through
    ``obg_detect_host``: the frames are staged into pinned memory by the
    native copy pool and moved with asynchronous copies pipelined around the
    classify kernel (a pageable ``cudaMemcpy`` of a frame is a single host
    thread at ~12 GB/s; per 1080p frame 0.83 -> see tools/sig_probe.py)."""
    frames = np.ascontiguousarray(frames)
    n, h, w = frames.shape[0], frames.shape[1], frames.shape[2]
    cfg = model.config
    cube = model.device_cube()
    out = np.empty((n, h, w), dtype=np.bool_)
    _lib.check(_lib.load().obg_detect_host(frames.ctypes.data, n, h, w, cfg.levels, cfg.grid_rows, cfg.grid_cols,
                                           _device.ptr(cube), out.ctypes.data, _device.stream_handle()))
    return out


def detect_octree(model: BackgroundModel, frame) -> np.ndarray:
    """Mask of pixels whose quantized colour is missing from their region's
    tree (detect.py:22-53).  A CUDA tensor in gives a CUDA bool tensor out."""
    if _device.is_tensor(frame):
        t = _device.torch()
        if frame.ndim != 3 or frame.shape[2] != 3 or frame.dtype != t.uint8:
            raise ValueError(f"expected (h, w, 3) uint8 frame, got {frame.dtype} {tuple(frame.shape)}")
        _check_frame_shape(model, int(frame.shape[0]), int(frame.shape[1]))
        _device.require_cuda()
        mask = classify(model, _device.to_device_u8(frame).unsqueeze(0))
        return mask[0].view(t.bool) if frame.is_cuda else mask[0].view(t.bool).cpu()
    frame = np.asarray(frame)
    if frame.ndim != 3 or frame.shape[2] != 3 or frame.dtype != np.uint8:
        raise ValueError(f"expected (h, w, 3) uint8 frame, got {frame.dtype} {frame.shape}")
    h, w = frame.shape[0], frame.shape[1]
    _check_frame_shape(model, h, w)
    _device.require_cuda()
    return _detect_host(model, frame[None])[0]


def detect_octree_batch(model: BackgroundModel, frames) -> np.ndarray:
    """``detect_octree`` over a (n, h, w, 3) batch in one launch -> (n, h, w) bool."""
    if _device.is_tensor(frames):
        mask = classify(model, frames)
        return mask.view(_device.torch().bool)
    frames = np.asarray(frames)
    if frames.ndim != 4 or frames.shape[3] != 3 or frames.dtype != np.uint8:
        raise ValueError(f"expected (n, h, w, 3) uint8 frames, got {frames.dtype} {frames.shape}")
    _check_frame_shape(model, frames.shape[1], frames.shape[2])
    _device.require_cuda()
    return _detect_host(model, frames)


# ---------------------------------------------------------------------------
# Comparison baselines (reference detect.py:56-83): frame difference and the
# running-mean background, on the GPU (obg_frame_diff / obg_running_average).
# ---------------------------------------------------------------------------
def _check_pair(a_shape, b_shape, what: str) -> None:
    """detect.py:17-19, same message."""
    if tuple(a_shape[:2]) != tuple(b_shape[:2]):
        raise ValueError(f"{what}: dimensions {tuple(a_shape[:2])} vs {tuple(b_shape[:2])} do not match")


def _check_u8_frames(x, what: str, batched: bool) -> None:
    nd = 4 if batched else 3
    shape = tuple(x.shape)
    dtype_ok = (x.dtype == _device.torch().uint8) if _device.is_tensor(x) else (x.dtype == np.uint8)
    if len(shape) != nd or shape[-1] != 3 or not dtype_ok:
        raise ValueError(f"{what}: expected {'(n, h, w, 3)' if batched else '(h, w, 3)'} uint8 frames, "
                         f"got {x.dtype} {shape}")


def frame_diff_sequence(frames_dev, diff_threshold: int = 30, out=None):
    """Masks of consecutive frame pairs of a (n, h, w, 3) uint8 CUDA tensor:
    mask t (t = 0..n-2) = detect_frame_diff(frames[t], frames[t + 1]) as 0/1
    bytes, ``(n - 1, h, w)`` uint8 CUDA tensor.  Every frame is read once."""
    _check_u8_frames(frames_dev, "frame difference", batched=True)
    frames_dev = _device.to_device_u8(frames_dev)
    n, h, w = int(frames_dev.shape[0]), int(frames_dev.shape[1]), int(frames_dev.shape[2])
    shape = (max(n - 1, 0), h, w)
    if out is None:
        out = _device.empty(shape, "uint8")
    elif tuple(out.shape) != shape or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous {shape} uint8 tensor")
    if n >= 2:
        p = _device.ptr(frames_dev)
        _lib.check(_lib.load().obg_frame_diff(p, p + 3 * h * w, n - 1, h * w, int(diff_threshold),
                                              _device.ptr(out), _device.stream_handle()))
    return out


def detect_frame_diff(previous, current, diff_threshold: int = 30):
    """Foreground where any channel changed by strictly more than the
    threshold (detect.py:56-63).  numpy in -> (h, w) bool numpy out; CUDA
    tensors in -> CUDA bool tensor out."""
    _check_pair(previous.shape, current.shape, "frame difference")
    _check_u8_frames(previous, "frame difference", batched=False)
    _check_u8_frames(current, "frame difference", batched=False)
    _device.require_cuda()
    a = _device.to_device_u8(previous if _device.is_tensor(previous) else np.asarray(previous))
    b = _device.to_device_u8(current if _device.is_tensor(current) else np.asarray(current))
    h, w = int(a.shape[0]), int(a.shape[1])
    out = _device.empty((h, w), "uint8")
    _lib.check(_lib.load().obg_frame_diff(_device.ptr(a), _device.ptr(b), 1, h * w, int(diff_threshold),
                                          _device.ptr(out), _device.stream_handle()))
    t = _device.torch()
    if _device.is_tensor(current) and current.is_cuda:
        return out.view(t.bool)
    return out.cpu().numpy().view(np.bool_)


def running_average_sequence(frames_dev, average_dev, frames_seen: int, diff_threshold: int = 30, out=None):
    """``detect_running_average`` over the frames of a (n, h, w, 3) uint8 CUDA
    tensor in one launch: returns the (n, h, w) uint8 0/1 masks and updates
    ``average_dev`` (a contiguous (h, w, 3) float64 CUDA tensor, the mean of
    the ``frames_seen`` frames already consumed) in place, bit-identical to
    calling the reference once per frame."""
    _check_u8_frames(frames_dev, "running average", batched=True)
    t = _device.torch()
    if not (_device.is_tensor(average_dev) and average_dev.is_cuda and average_dev.dtype == t.float64
            and average_dev.is_contiguous() and average_dev.ndim == 3 and average_dev.shape[2] == 3):
        raise ValueError("average must be a contiguous (h, w, 3) float64 CUDA tensor")
    _check_pair(average_dev.shape, frames_dev.shape[1:], "running average")
    frames_dev = _device.to_device_u8(frames_dev)
    n, h, w = int(frames_dev.shape[0]), int(frames_dev.shape[1]), int(frames_dev.shape[2])
    if out is None:
        out = _device.empty((n, h, w), "uint8")
    elif tuple(out.shape) != (n, h, w) or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous {(n, h, w)} uint8 tensor")
    _lib.check(_lib.load().obg_running_average(_device.ptr(frames_dev), n, h * w, int(frames_seen),
                                               _device.ptr(average_dev), int(diff_threshold), _device.ptr(out),
                                               _device.stream_handle()))
    return out


def detect_running_average(frames_seen: int, average, current, diff_threshold: int = 30):
    """One step of the running-mean baseline (detect.py:66-83): returns the
    mask of ``current`` against the float64 mean of the ``frames_seen``
    frames already consumed, and the mean updated to include ``current``
    (IEEE binary64, bit-identical to the reference)."""
    average = np.asarray(average, dtype=np.float64)
    _check_pair(average.shape, current.shape, "running average")
    _check_u8_frames(current, "running average", batched=False)
    if average.ndim != 3 or average.shape[2] != 3:
        raise ValueError(f"running average: expected a (h, w, 3) mean, got {average.shape}")
    _device.require_cuda()
    t = _device.torch()
    avg = t.from_numpy(np.ascontiguousarray(average)).to("cuda")
    frame = _device.to_device_u8(current if _device.is_tensor(current) else np.asarray(current))
    masks = running_average_sequence(frame.unsqueeze(0), avg, frames_seen, diff_threshold)
    return masks[0].cpu().numpy().view(np.bool_), avg.cpu().numpy()
