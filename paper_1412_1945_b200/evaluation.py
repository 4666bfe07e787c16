"""Confusion counts and the negative-oriented F0 score, with classification
fused into the counting on the device.

Host names and semantics follow the reference's ``evaluation.py``:
``EvalStats`` (evaluation.py:16-35; foreground is the positive class, fields
in the order tn, tp, fn, fp), ``accumulate`` (38-53), ``f0_score`` (56-70,
P0 = Tn/(Tn+Fn), R0 = Tn/(Tn+Fp), None when a denominator is zero) and
``emit_report`` (76-84).  ``classify_confusion`` is the device path: one
launch classifies a batch of frames and counts it against ground-truth masks
without writing a mask (``obg_classify_confusion``), so evaluating costs the
classify bandwidth plus one byte (or bit) of truth per pixel.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device, _lib
from .model import BackgroundModel


@dataclass(frozen=True)
class EvalStats:
    """Pixel confusion counts; foreground is the positive class."""

    true_neg: int = 0
    true_pos: int = 0
    false_neg: int = 0
    false_pos: int = 0

    def __add__(self, other: "EvalStats") -> "EvalStats":
        return EvalStats(self.true_neg + other.true_neg, self.true_pos + other.true_pos,
                         self.false_neg + other.false_neg, self.false_pos + other.false_pos)

    @property
    def total(self) -> int:
        return self.true_neg + self.true_pos + self.false_neg + self.false_pos


def accumulate(predicted, truth, stats: EvalStats | None = None) -> EvalStats:
    """``stats`` plus the confusion counts of one predicted / truth mask pair."""
    if _device.is_tensor(predicted) or _device.is_tensor(truth):
        t = _device.torch()
        p = predicted.bool() if _device.is_tensor(predicted) else t.from_numpy(np.asarray(predicted, bool))
        g = truth.bool() if _device.is_tensor(truth) else t.from_numpy(np.asarray(truth, bool))
        if tuple(p.shape) != tuple(g.shape):
            raise ValueError(f"mask dimensions {tuple(p.shape)} vs {tuple(g.shape)} do not match")
        g = g.to(p.device)
        counts = [int(x) for x in ((~p & ~g).sum(), (p & g).sum(), (~p & g).sum(), (p & ~g).sum())]
    else:
        p = np.asarray(predicted, dtype=bool)
        g = np.asarray(truth, dtype=bool)
        if p.shape != g.shape:
            raise ValueError(f"mask dimensions {p.shape} vs {g.shape} do not match")
        counts = [int(np.count_nonzero(~p & ~g)), int(np.count_nonzero(p & g)),
                  int(np.count_nonzero(~p & g)), int(np.count_nonzero(p & ~g))]
    return (stats if stats is not None else EvalStats()) + EvalStats(*counts)


def f0_score(stats: EvalStats):
    """(P0, R0, F0); an undefined ratio is None, never a made-up zero."""
    tn, fn, fp = stats.true_neg, stats.false_neg, stats.false_pos
    p0 = tn / (tn + fn) if tn + fn > 0 else None
    r0 = tn / (tn + fp) if tn + fp > 0 else None
    f0 = None if p0 is None or r0 is None or p0 + r0 == 0 else 2 * p0 * r0 / (p0 + r0)
    return p0, r0, f0


def _fmt(score) -> str:
    return "undefined" if score is None else f"{score:.6f}"


def emit_report(rows) -> str:
    """CSV table: one line per (method, dataset, stats), in input order."""
    out = ["method,dataset,tn,tp,fn,fp,p0,r0,f0"]
    for method, dataset, s in rows:
        p0, r0, f0 = f0_score(s)
        out.append(f"{method},{dataset},{s.true_neg},{s.true_pos},{s.false_neg},{s.false_pos},"
                   f"{_fmt(p0)},{_fmt(r0)},{_fmt(f0)}")
    return "\n".join(out) + "\n"


def classify_confusion(model: BackgroundModel, frames_dev, truth_dev, stats: EvalStats | None = None,
                       packed: bool = False) -> EvalStats:
    """``stats`` plus the confusion counts of ``detect_octree`` on every frame
    of a (n, h, w, 3) uint8 CUDA tensor against ``truth_dev``, in one fused
    launch (no mask is materialised).

    ``truth_dev``: CUDA tensor (n, h, w) of bool / uint8 (nonzero =
    foreground, so 0/255 PGM values work as read), or with ``packed`` the
    (n, ceil(h*w/8)) LSB-first bit layout of ``classify(..., packed=True)``.
    """
    from .detect import _check_frame_shape
    t = _device.torch()
    frames_dev = _device.frames_on_device(frames_dev)
    n, h, w = int(frames_dev.shape[0]), int(frames_dev.shape[1]), int(frames_dev.shape[2])
    _check_frame_shape(model, h, w)
    want = (n, (h * w + 7) // 8) if packed else (n, h, w)
    if tuple(truth_dev.shape) != want:
        raise ValueError(f"mask dimensions {tuple(truth_dev.shape)} vs {want} do not match")
    truth = truth_dev.view(t.uint8) if truth_dev.dtype == t.bool else truth_dev
    if truth.dtype != t.uint8:
        raise ValueError(f"expected a bool or uint8 truth mask, got {truth_dev.dtype}")
    truth = truth.to(frames_dev.device).contiguous()
    cfg = model.config
    counts = t.zeros(4, dtype=t.int64, device=frames_dev.device)
    lib = _lib.load()
    _lib.check(lib.obg_classify_confusion(
        _device.ptr(frames_dev), n, h, w, cfg.levels, cfg.grid_rows, cfg.grid_cols,
        _device.ptr(model.device_cube()), _device.ptr(truth), _lib.MASK_PACKED if packed else _lib.MASK_U8,
        _device.ptr(counts), _device.stream_handle()))
    got = EvalStats(*[int(x) for x in counts.cpu().tolist()])
    return (stats if stats is not None else EvalStats()) + got
