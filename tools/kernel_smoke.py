"""Small run of every kernel family and entry point (L 2..8, 1x1 and 2x3
grids, odd frame sizes, sharded build, baselines) -- a launch smoke test.

    python tools/sanitize_probe.py      (GPU box)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_1945_b200 as obg  # noqa: E402
from paper_1412_1945_b200.distributed import build_background_model_sharded  # noqa: E402

rng = np.random.default_rng(5)
h, w = 48, 64
base = rng.integers(0, 256, size=(1, h, w, 3))
frames = np.clip(base + rng.integers(-30, 31, size=(6, h, w, 3)), 0, 255).astype(np.uint8)
dev = torch.from_numpy(frames).cuda()
odd = torch.from_numpy(np.ascontiguousarray(frames[:, :45, :61])).cuda()
for L in (2, 4, 5, 6, 7, 8):
    for grid in ((1, 1), (2, 3)):
        cfg = obg.ModelConfig(levels=L, threshold=0.5, grid_rows=grid[0], grid_cols=grid[1], training_frames=6)
        m = obg.build_background_model_device(dev, cfg)
        obg.classify(m, dev)
        obg.classify(m, dev, packed=True)
        obg.classify_confusion(m, dev, torch.zeros(dev.shape[:3], dtype=torch.uint8, device="cuda"))
        m.trees[0][0].to_bytes()
        build_background_model_sharded(dev, cfg)
        obg.build_presence(dev, L, grid[0], grid[1], 2)
        mo = obg.build_background_model_device(odd, cfg)
        obg.classify(mo, odd)
obg.frame_diff_sequence(dev, 30)
obg.running_average_sequence(dev, dev[0].to(torch.float64).contiguous(), 1, 30)
torch.cuda.synchronize()
print("kernel smoke done")
