"""Pinned H2D / D2H time against transfer size (GPU box)."""
import time
import torch

def t(fn, reps=7):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1000

for mb in (0.25, 1, 2, 6.2, 12, 25, 50, 100, 400):
    n = int(mb * 1e6)
    pin = torch.empty(n, dtype=torch.uint8).pin_memory()
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    h = t(lambda: dev.copy_(pin, non_blocking=True))
    d = t(lambda: pin.copy_(dev, non_blocking=True))
    # split into 4 async copies on 2 streams
    s = [torch.cuda.Stream() for _ in range(4)]
    q = n // 4
    def split():
        for i in range(4):
            with torch.cuda.stream(s[i]):
                dev[i * q:(i + 1) * q].copy_(pin[i * q:(i + 1) * q], non_blocking=True)
    sp = t(split)
    print(f"{mb:7.2f} MB  H2D {h:7.3f} ms {n / h / 1e6:6.1f} GB/s   D2H {d:7.3f} ms {n / d / 1e6:6.1f} GB/s   H2D 4 streams {sp:7.3f} ms {n / sp / 1e6:6.1f} GB/s")
