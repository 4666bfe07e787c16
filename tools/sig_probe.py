"""Where the literal reference-signature e2e goes (GPU box): list of numpy
frames -> build_background_model, then detect_octree per numpy frame."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_1945_b200 as obg  # noqa: E402
from paper_1412_1945_b200 import scenes  # noqa: E402


def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1000


sc = scenes.generate(3, n_test=32)
train, test = list(sc.train), list(sc.test)
cfg = obg.ModelConfig(levels=6, threshold=0.5, training_frames=64)
model = obg.build_background_model(train, cfg)
print(f"np.stack 64 frames        {t(lambda: np.stack(train)):8.2f} ms")
st = np.stack(train)
print(f"H2D pageable 64 frames    {t(lambda: torch.from_numpy(st).to('cuda')):8.2f} ms")
print(f"build_background_model    {t(lambda: obg.build_background_model(train, cfg)):8.2f} ms")
f = test[0]
print(f"detect_octree x32         {t(lambda: [obg.detect_octree(model, x) for x in test]) / 32:8.3f} ms/frame")
print(f"  H2D pageable 1 frame    {t(lambda: torch.from_numpy(f).to('cuda')):8.3f} ms")
dev = torch.from_numpy(f[None]).cuda()
print(f"  classify 1 frame        {t(lambda: obg.classify(model, dev)):8.3f} ms")
m = obg.classify(model, dev)
print(f"  D2H pageable mask       {t(lambda: m.cpu()):8.3f} ms")
pin = torch.empty(f.shape, dtype=torch.uint8).pin_memory()
print(f"  copy into pinned        {t(lambda: pin.numpy().__setitem__(Ellipsis, f)):8.3f} ms")
