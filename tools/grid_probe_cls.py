import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1412_1945_b200 as obg  # noqa: E402
from kbench import frames_for, timeit  # noqa: E402
f = torch.from_numpy(frames_for("c3", 64, 6)).cuda()
for grid in ((2, 2), (3, 4)):
    cfg = obg.ModelConfig(levels=6, threshold=0.5, grid_rows=grid[0], grid_cols=grid[1], training_frames=64)
    model = obg.build_background_model_device(f, cfg)
    out = torch.empty(f.shape[:3], dtype=torch.uint8, device="cuda")
    print(f"grid {grid}: classify: {timeit(lambda: obg.classify(model, f, out=out)) * 1000:.1f} us")
