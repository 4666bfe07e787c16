"""Per-frame cost of detect_octree (numpy in / out) through obg_detect_host, against the
pageable-copy path it replaced, and the pieces (GPU box)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_1945_b200 as obg  # noqa: E402
from paper_1412_1945_b200 import scenes, _device  # noqa: E402


def t(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1000


sc = scenes.generate(3, n_train=16, n_test=32)
train, test = list(sc.train), list(sc.test)
cfg = obg.ModelConfig(levels=6, threshold=0.5, training_frames=16)
model = obg.build_background_model(train, cfg)


def old_path(x):
    mask = obg.classify(model, _device.to_device_u8(x[None]))
    return mask[0].cpu().numpy().view(np.bool_)


ref = [old_path(x) for x in test]
new = [obg.detect_octree(model, x) for x in test]
print("equal:", all(np.array_equal(a, b) for a, b in zip(ref, new)))
print(f"pageable path   x32  {t(lambda: [old_path(x) for x in test]) / 32:8.3f} ms/frame")
print(f"detect_octree   x32  {t(lambda: [obg.detect_octree(model, x) for x in test]) / 32:8.3f} ms/frame")
st = np.stack(test)
print(f"detect_octree_batch(32 numpy frames) {t(lambda: obg.detect_octree_batch(model, st)) / 32:8.3f} ms/frame")
pin = torch.empty(test[0].shape, dtype=torch.uint8).pin_memory()
print(f"  pool copy 1 frame -> pinned {t(lambda: _device.host_gather([test[0]], pin.data_ptr(), test[0].nbytes)):8.3f} ms")
dev = torch.empty(test[0].shape, dtype=torch.uint8, device='cuda')
print(f"  H2D pinned 1 frame          {t(lambda: dev.copy_(pin, non_blocking=True)):8.3f} ms")
