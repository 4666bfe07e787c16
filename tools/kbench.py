"""Micro-benchmark of individual kernels on synthetic inputs (CUDA events).

    python tools/kbench.py build|model|classify|confusion [--frames N] [--scene c3|const|repeat|uniform] [--levels L]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_1945_b200 as obg  # noqa: E402
from paper_1412_1945_b200 import scenes  # noqa: E402


def frames_for(kind, n, levels):
    cache = f"/tmp/kbench_{kind}_{n}_{levels}.npy"      # A/B runs (tools/ab.py) reuse the frames
    if os.path.exists(cache):
        return np.load(cache)
    f = _frames_for(kind, n, levels)
    try:
        np.save(cache, f)
    except OSError:
        pass
    return f


def _frames_for(kind, n, levels):
    if kind in ("c0", "c1", "c2", "c3"):          # BASELINE configs 0..3 scenes
        return scenes.generate(int(kind[1]), n_train=n, n_test=0).train
    if kind == "const":
        f = np.empty((n, 1080, 1920, 3), np.uint8)
        f[...] = (90, 140, 60)
        return f
    if kind == "repeat":
        one = scenes.generate(3, n_train=1, n_test=0).train
        return np.repeat(one, n, axis=0)
    if kind in ("c4uniform", "c4constant"):       # BASELINE config 4 (3840x2160) scenes
        return scenes.generate(4, n_train=n, n_test=0, levels=levels, variant=kind[2:]).train
    if kind == "uniform":
        return np.random.default_rng(0).integers(0, 256, size=(n, 1080, 1920, 3), dtype=np.uint8)
    raise SystemExit(kind)


GRAPH = "--graph" in sys.argv


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    if GRAPH:          # device time without the host launch overhead: one captured call, replayed
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        fn = g.replay
        fn()
        torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["build", "counts", "classify", "model", "sharded", "confusion", "framediff", "runavg"])
    ap.add_argument("--frames", type=int, default=64)
    ap.add_argument("--scene", default="c3")
    ap.add_argument("--levels", type=int, default=6)
    ap.add_argument("--threshold", type=float, default=0.5)
    ap.add_argument("--graph", action="store_true", help="time CUDA-graph replays (no host launch overhead)")
    a = ap.parse_args()
    f = torch.from_numpy(frames_for(a.scene, a.frames, a.levels)).cuda()
    px = f.shape[0] * f.shape[1] * f.shape[2]
    cfg = obg.ModelConfig(levels=a.levels, threshold=a.threshold, training_frames=a.frames)
    digest = ""
    if a.what == "build":
        ms = timeit(lambda: obg.build_presence(f, a.levels))
    elif a.what == "counts":         # presence + a13 occupancy counts (k_hist pass)
        ms = timeit(lambda: obg.build_presence(f, a.levels, counts=True))
        import hashlib
        digest = " model=" + hashlib.sha1(obg.build_presence(f, a.levels, counts=True)[1].cpu().numpy().tobytes()).hexdigest()[:12]
    elif a.what == "model":
        ms = timeit(lambda: obg.build_background_model_device(f, cfg))
        m = obg.build_background_model_device(f, cfg)
        import hashlib
        h = hashlib.sha1(m._dev_pyr.cpu().numpy().tobytes())
        h.update(m._dev_cube.cpu().numpy().tobytes())
        digest = " model=" + h.hexdigest()[:12]
    elif a.what == "confusion":      # fused classify + evaluation against a truth mask (4 B/px)
        model = obg.build_background_model_device(f, cfg)
        truth = (torch.rand(f.shape[:3], device="cuda") < 0.3).to(torch.uint8)
        ms = timeit(lambda: obg.classify_confusion(model, f, truth))
    elif a.what == "sharded":        # the multi-GPU build path (counts + threshold), no process group
        from paper_1412_1945_b200.distributed import build_background_model_sharded
        ms = timeit(lambda: build_background_model_sharded(f, cfg))
    elif a.what == "framediff":      # consecutive-pair masks, every frame read once (4 B/px)
        out = torch.empty((f.shape[0] - 1,) + tuple(f.shape[1:3]), dtype=torch.uint8, device="cuda")
        ms = timeit(lambda: obg.frame_diff_sequence(f, 30, out=out))
    elif a.what == "runavg":         # running mean over the batch: 4 B/px per frame + 48 B/px per call
        avg = f[0].to(torch.float64).contiguous()
        out = torch.empty(f.shape[:3], dtype=torch.uint8, device="cuda")
        ms = timeit(lambda: obg.running_average_sequence(f, avg, 1, 30, out=out))
    else:
        model = obg.build_background_model_device(f, cfg)
        out = torch.empty(f.shape[:3], dtype=torch.uint8, device="cuda")
        ms = timeit(lambda: obg.classify(model, f, out=out))
    print(f"{a.what} scene={a.scene} L={a.levels} frames={a.frames}: {ms * 1000:.1f} us, "
          f"{px / ms / 1e6:.1f} Gpx/s, {px * (4 if a.what in ('classify', 'confusion', 'framediff', 'runavg') else 3) / ms / 1e6:.1f} GB/s{digest}")


if __name__ == "__main__":
    main()
