"""Seeded synthetic scenes with the shapes of BASELINE.json's five configs.

The paper's Wallflower sequences are not available (and the reference's own
``synth.py`` implements different scenes), so these generators stand in for
them: same frame sizes, octree depths, frame counts, thresholds and the value
distributions BASELINE.json describes (gradient + Gaussian noise, brightness
ramp, bimodal "swaying" region, moving rectangles / ellipses, uniform-random
and constant stress frames).

Every frame is produced from its own ``numpy.random.default_rng`` stream keyed
by (seed, config, split, index), so frame i is identical whether a caller asks
for 10 frames or 256 -- bounded CPU samples and full GPU batches see the same
pixels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .model import ModelConfig

# (width, height, levels, n_train, n_test, threshold)
CONFIGS = {
    0: (160, 120, 4, 20, 10, 0.5),
    1: (640, 480, 5, 30, 100, 0.5),
    2: (1280, 720, 5, 50, 200, 0.3),
    3: (1920, 1080, 6, 64, 256, 0.5),
    4: (3840, 2160, 6, 32, 128, 0.5),   # levels swept 4..7 by the caller
}
NAMES = {0: "C0 160x120 L4", 1: "C1 640x480 L5", 2: "C2 1280x720 L5", 3: "C3 1920x1080 L6",
         4: "C4 3840x2160 stress"}


@dataclass
class Scene:
    config_id: int
    variant: str
    config: ModelConfig
    width: int
    height: int
    train: np.ndarray   # (n_train, h, w, 3) uint8
    test: np.ndarray    # (n_test, h, w, 3) uint8


def _rng(seed: int, cfg: int, split: int, index: int) -> np.random.Generator:
    return np.random.default_rng([seed, cfg, split, index])


class _SceneParams:
    def __init__(self, cfg: int, seed: int, width: int, height: int, n_train: int, n_test: int):
        rng = _rng(seed, cfg, 9, 0)
        self.cfg, self.w, self.h = cfg, width, height
        self.total = n_train_full(cfg) + n_test_full(cfg)
        lo = rng.uniform(20, 110, size=3)
        hi = rng.uniform(140, 235, size=3)
        xs = np.linspace(0.0, 1.0, width, dtype=np.float32)
        ys = np.linspace(0.0, 1.0, height, dtype=np.float32)
        ramp = [xs[None, :] + 0 * ys[:, None], ys[:, None] + 0 * xs[None, :],
                0.5 * (xs[None, :] + ys[:, None])]
        self.bg = np.stack([(lo[c] + (hi[c] - lo[c]) * ramp[c]).astype(np.float32) for c in range(3)], axis=-1)
        self.sway_rows = int(round(0.2 * height))
        self.sway_colors = rng.integers(0, 256, size=(2, 3)).astype(np.float32)
        self.const_color = rng.integers(0, 256, size=3).astype(np.uint8)
        # moving objects: position, velocity, size, colour
        n_obj = {1: 5, 2: 8, 3: 8}.get(cfg, 0)
        self.objects = []
        for _ in range(n_obj):
            if cfg == 1:
                size = rng.integers(8, 41, size=2)
            else:
                size = rng.integers(max(8, height // 40), max(16, height // 8), size=2)
            pos = rng.uniform(0, 1, size=2) * np.array([width - size[0], height - size[1]])
            speed = rng.uniform(2, 6, size=2) * rng.choice([-1.0, 1.0], size=2)
            colour = rng.integers(0, 256, size=3).astype(np.uint8)
            self.objects.append((pos, speed, size, colour))
        n_boot = int(round(0.1 * n_train_full(cfg))) if cfg == 3 else 0
        self.bootstrap = set(rng.choice(n_train_full(cfg), size=n_boot, replace=False).tolist()) if n_boot else set()


def n_train_full(cfg: int) -> int:
    return CONFIGS[cfg][3]


def n_test_full(cfg: int) -> int:
    return CONFIGS[cfg][4]


def _bounce(p: float, v: float, t: int, span: float) -> float:
    if span <= 0:
        return 0.0
    x = (p + v * t) % (2 * span)
    return x if x <= span else 2 * span - x


def _draw_rects(frame: np.ndarray, rng: np.random.Generator, lo: int, hi: int) -> None:
    h, w = frame.shape[:2]
    for _ in range(int(rng.integers(lo, hi + 1))):
        rw, rh = (int(v) for v in rng.integers(8, 41, size=2))
        x = int(rng.integers(0, max(1, w - rw)))
        y = int(rng.integers(0, max(1, h - rh)))
        frame[y:y + rh, x:x + rw] = rng.integers(0, 256, size=3).astype(np.uint8)


def _frame(p: _SceneParams, seed: int, variant: str, split: int, index: int) -> np.ndarray:
    rng = _rng(seed, p.cfg, split, index)
    t = index if split == 0 else n_train_full(p.cfg) + index      # global time
    if p.cfg == 4:
        if variant == "uniform":
            frame = rng.integers(0, 256, size=(p.h, p.w, 3), dtype=np.uint8)
        else:
            frame = np.empty((p.h, p.w, 3), dtype=np.uint8)
            frame[...] = p.const_color
        if split == 1:
            _draw_rects(frame, rng, 1, 3)
        return frame
    f = p.bg.copy()
    if p.cfg == 1:
        f += np.float32(-10.0 + 20.0 * t / max(1, p.total - 1))
    f += rng.standard_normal(size=f.shape, dtype=np.float32) * np.float32(3.0)
    if p.cfg in (2, 3):
        sr = p.sway_rows
        pick = rng.random(size=(sr, p.w)) < 0.5
        sway = np.where(pick[..., None], p.sway_colors[0], p.sway_colors[1])
        f[:sr] = sway + rng.standard_normal(size=sway.shape, dtype=np.float32) * np.float32(3.0)
    frame = np.clip(np.rint(f), 0, 255).astype(np.uint8)
    if split == 1 or index in p.bootstrap:
        if p.cfg == 0 or split == 0:
            _draw_rects(frame, rng, 1, 3)
        elif p.cfg == 1:
            for pos, speed, size, colour in p.objects:
                x = int(_bounce(pos[0], speed[0], t, p.w - size[0]))
                y = int(_bounce(pos[1], speed[1], t, p.h - size[1]))
                frame[y:y + size[1], x:x + size[0]] = colour
        else:
            yy, xx = np.ogrid[:p.h, :p.w]
            for pos, speed, size, colour in p.objects:
                ax, ay = size[0] / 2.0, size[1] / 2.0
                cx = _bounce(pos[0], speed[0], t, p.w - size[0]) + ax
                cy = _bounce(pos[1], speed[1], t, p.h - size[1]) + ay
                y0, y1 = max(0, int(cy - ay)), min(p.h, int(cy + ay) + 1)
                x0, x1 = max(0, int(cx - ax)), min(p.w, int(cx + ax) + 1)
                sub = ((xx[:, x0:x1] - cx) / ax) ** 2 + ((yy[y0:y1] - cy) / ay) ** 2 <= 1.0
                frame[y0:y1, x0:x1][sub] = colour
    return frame


def generate(config_id: int, seed: int = 1412, n_train: int | None = None, n_test: int | None = None,
             levels: int | None = None, variant: str = "uniform") -> Scene:
    """Frames of BASELINE config ``config_id`` (0..4).  ``n_train`` / ``n_test``
    take a prefix of the full sequence; ``levels`` overrides the depth (config
    4 sweeps 4..7); ``variant`` selects config 4's "uniform" or "constant"
    background."""
    width, height, lv, nt, ns, thr = CONFIGS[config_id]
    n_train = nt if n_train is None else n_train
    n_test = ns if n_test is None else n_test
    levels = lv if levels is None else levels
    if config_id != 4:
        variant = "natural"
    p = _SceneParams(config_id, seed, width, height, n_train, n_test)
    train = np.empty((n_train, height, width, 3), dtype=np.uint8)
    test = np.empty((n_test, height, width, 3), dtype=np.uint8)
    for i in range(n_train):
        train[i] = _frame(p, seed, variant, 0, i)
    for i in range(n_test):
        test[i] = _frame(p, seed, variant, 1, i)
    cfg = ModelConfig(levels=levels, threshold=thr, training_frames=max(1, n_train))
    return Scene(config_id, variant, cfg, width, height, train, test)
