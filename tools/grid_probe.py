"""Time the model build and classify with a region grid (generic kernels) vs 1x1 (GPU box)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1412_1945_b200 as obg  # noqa: E402
from kbench import frames_for, timeit  # noqa: E402

f = torch.from_numpy(frames_for("c3", 64, 6)).cuda()
for grid in ((1, 1), (2, 2), (3, 4)):
    cfg = obg.ModelConfig(levels=6, threshold=0.5, grid_rows=grid[0], grid_cols=grid[1], training_frames=64)
    ms_b = timeit(lambda: obg.build_background_model_device(f, cfg))
    model = obg.build_background_model_device(f, cfg)
    out = torch.empty(f.shape[:3], dtype=torch.uint8, device="cuda")
    ms_c = timeit(lambda: obg.classify(model, f, out=out))
    px = f.shape[0] * f.shape[1] * f.shape[2]
    print(f"grid {grid}: build {ms_b * 1000:.1f} us ({px * 3 / ms_b / 1e6:.0f} GB/s), "
          f"classify {ms_c * 1000:.1f} us ({px * 4 / ms_c / 1e6:.0f} GB/s)")
