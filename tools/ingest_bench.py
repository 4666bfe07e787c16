"""Ingest pipeline throughput (GPU box): PPM directory -> pinned frames ->
model + masks (pipeline.detect_sequence), against the per-file Python reader.

    python tools/ingest_bench.py [--frames 128] [--dir /tmp/obg_ingest]

Files are freshly written, so they are read from the page cache: this
measures parsing + copying into pinned memory + the GPU pipeline, not disk.
"""
import argparse
import os
import shutil
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_1945_b200 as obg  # noqa: E402
from paper_1412_1945_b200 import pipeline, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=128)
    ap.add_argument("--dir", default="/tmp/obg_ingest")
    a = ap.parse_args()
    sc = scenes.generate(3, n_train=64, n_test=max(0, a.frames - 64))
    frames = np.concatenate([sc.train, sc.test])[: a.frames]
    shutil.rmtree(a.dir, ignore_errors=True)
    seq = obg.write_frame_sequence(os.path.join(a.dir, "frames"), list(frames))
    px = frames.shape[0] * frames.shape[1] * frames.shape[2]
    out = torch.empty((len(seq), seq.height, seq.width, 3), dtype=torch.uint8, pin_memory=True)
    seq.load_batch(out=out)                                  # page-in
    t0 = time.perf_counter()
    seq.load_batch(out=out)
    t1 = time.perf_counter()
    seq.load_all()
    t2 = time.perf_counter()
    cfg = obg.ModelConfig(levels=6, threshold=0.5, training_frames=64)
    pipeline.detect_sequence(seq, cfg)                       # warm-up
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    _, masks = pipeline.detect_sequence(seq, cfg)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    pipeline.detect_sequence(seq, cfg, out_dir=os.path.join(a.dir, "masks"))
    t5 = time.perf_counter()
    gb = frames.nbytes / 1e9
    print(f"load_batch (threads, pinned): {gb / (t1 - t0):.2f} GB/s; per-file load_all: {gb / (t2 - t1):.2f} GB/s")
    print(f"detect_sequence -> host masks: {px / (t4 - t3) / 1e6:.0f} Mpx/s ({a.frames / (t4 - t3):.0f} frames/s)")
    print(f"detect_sequence -> PGM files:  {px / (t5 - t4) / 1e6:.0f} Mpx/s ({a.frames / (t5 - t4):.0f} frames/s)")
    shutil.rmtree(a.dir, ignore_errors=True)


if __name__ == "__main__":
    main()
