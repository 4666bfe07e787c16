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


def classify(model: BackgroundModel, frames_dev, out=None, packed: bool = False):
    """Foreground masks of a (n, h, w, 3) uint8 CUDA tensor.

    Returns (and fills ``out`` if given) a uint8 CUDA tensor: ``(n, h, w)``
    0/1 bytes, or ``(n, ceil(h*w/8))`` LSB-first bits when ``packed``.
    A pixel is foreground iff its quantized colour is not a full-depth leaf
    of its region's merged tree; an empty tree flags everything (detect.py:44-52).
    """
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
                                _lib.MASK_PACKED if packed else _lib.MASK_U8, _device.stream_handle()))
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
    _check_frame_shape(model, frame.shape[0], frame.shape[1])
    _device.require_cuda()
    mask = classify(model, _device.to_device_u8(frame[None]))
    return mask[0].cpu().numpy().view(np.bool_)


def detect_octree_batch(model: BackgroundModel, frames) -> np.ndarray:
    """``detect_octree`` over a (n, h, w, 3) batch in one launch -> (n, h, w) bool."""
    if _device.is_tensor(frames):
        mask = classify(model, _device.to_device_u8(frames))
        return mask.view(_device.torch().bool)
    frames = np.asarray(frames)
    if frames.ndim != 4 or frames.shape[3] != 3 or frames.dtype != np.uint8:
        raise ValueError(f"expected (n, h, w, 3) uint8 frames, got {frames.dtype} {frames.shape}")
    _check_frame_shape(model, frames.shape[1], frames.shape[2])
    _device.require_cuda()
    mask = classify(model, _device.to_device_u8(frames))
    return mask.cpu().numpy().view(np.bool_)
