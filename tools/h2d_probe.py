"""H2D bandwidth from pinned memory with 1, 2 and 4 concurrent copy streams (GPU box)."""
import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunk = n // k
    for rep in range(3):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for i, st in enumerate(streams):
            st.wait_event(s)
            with torch.cuda.stream(st):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for st in streams:
            torch.cuda.current_stream().wait_stream(st)
        e.record()
        torch.cuda.synchronize()
    print(f"{k} stream(s): H2D {n / s.elapsed_time(e) / 1e6:.1f} GB/s")
