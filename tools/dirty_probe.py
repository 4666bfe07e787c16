"""Does a pinned buffer that the CPU has just written (dirty lines in the CPU caches) DMA slower?"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1412_1945_b200 import _device

def once(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1000

n = 6220800
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
pin = torch.empty(n, dtype=torch.uint8).pin_memory()
src = np.random.default_rng(0).integers(0, 255, n, dtype=np.uint8)
big = np.zeros(512 << 20, np.uint8)
h2d = lambda: dev.copy_(pin, non_blocking=True)
for _ in range(3): once(h2d)
print("clean, repeated:", [round(once(h2d), 3) for _ in range(4)])
for trial in range(3):
    pin.numpy()[:] = src                      # single-thread memcpy into the pinned buffer
    a = once(h2d); b = once(h2d); c = once(h2d)
    print(f"after main-thread write: {a:.3f} {b:.3f} {c:.3f} ms")
for trial in range(3):
    _device.host_gather([src], pin.data_ptr(), n)   # pool threads write it
    a = once(h2d); b = once(h2d); c = once(h2d)
    print(f"after pool write:        {a:.3f} {b:.3f} {c:.3f} ms")
_device.host_gather([src], pin.data_ptr(), n)
big[:] = 1                                     # push the dirty lines out of the caches
print("after pool write + 512 MB cache sweep:", [round(once(h2d), 3) for _ in range(3)])
