"""Randomised GPU-vs-oracle fuzz of build / merge / classify / counts (GPU box).

    python tools/fuzz_gpu.py [seconds] [seed]

Shapes are drawn around the kernels' structural boundaries (16-pixel units,
1024-unit CTA iterations, tree segments), levels 1..8, grids, groups and
thresholds at random; every merged tree (to_bytes), every mask and the leaf
counts are compared with the CPU oracle (test infrastructure, oracle/).
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_1945_b200 as obg  # noqa: E402
from oracle import octree_oracle as orc  # noqa: E402


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
    t0, n = time.time(), 0
    while time.time() - t0 < budget:
        L = int(rng.integers(1, 9))
        kind = rng.integers(0, 4)
        if kind == 0:      # pixel counts around multiples of 16 * 1024
            px = int(rng.integers(1, 4)) * 16384 + int(rng.integers(-40, 41))
            w = int(rng.choice([16, 32, 48, 64, 128, 17, 100]))
            h = max(1, px // w)
        elif kind == 1:    # tiny / odd
            h, w = int(rng.integers(1, 40)), int(rng.integers(1, 70))
        else:
            h, w = int(rng.integers(8, 200)), 16 * int(rng.integers(1, 24))
        grid = (1, 1) if rng.random() < 0.6 else (int(rng.integers(1, 4)), int(rng.integers(1, 5)))
        grid = (min(grid[0], h), min(grid[1], w))
        gs = int(rng.choice([1, 1, 2, 3]))
        n_train = gs * int(rng.integers(1, 9)) + int(rng.integers(0, gs))
        thr = float(rng.choice([0.5, 0.3, 1.0, 0.55, 1.0 / max(1, n_train // gs), 0.26]))
        spread = int(rng.choice([2, 8, 40, 128]))
        base = rng.integers(0, 256, size=(1, 1, 1, 3))
        mk = lambda k: np.clip(base + rng.integers(-spread, spread + 1, size=(k, h, w, 3)), 0, 255).astype(np.uint8)
        if rng.random() < 0.15:
            mk = lambda k: rng.integers(0, 256, size=(k, h, w, 3), dtype=np.uint8)
        train, probe = mk(n_train), mk(2)
        cfg = obg.ModelConfig(levels=L, threshold=thr, grid_rows=grid[0], grid_cols=grid[1], group_size=gs,
                              training_frames=max(n_train, gs))
        tag = f"L={L} {h}x{w} grid={grid} gs={gs} n={n_train} thr={thr:.3f} spread={spread}"
        model = obg.build_background_model(list(train), cfg)
        want = orc.build_background_model(list(train), L, thr, grid[0], grid[1], gs)
        for r in range(grid[0]):
            for c in range(grid[1]):
                assert model.trees[r][c].to_bytes() == orc.to_bytes(want[(r, c)]), ("tree", tag, r, c)
        got = obg.detect_octree_batch(model, probe)
        for i in range(2):
            assert np.array_equal(got[i], orc.detect_octree(want, probe[i], L, grid[0], grid[1])), ("mask", tag, i)
        dev = obg.classify(model, torch.from_numpy(probe).cuda()).cpu().numpy().astype(bool)
        assert np.array_equal(dev, got), ("device mask", tag)
        if grid == (1, 1) and L <= 7:
            _, counts = obg.build_presence(torch.from_numpy(train).cuda(), L, counts=True)
            c0 = counts[0, 0].cpu().numpy().reshape(-1)
            ref = np.bincount(orc.pack_codes(train[0], L).ravel(), minlength=8 ** L)
            assert np.array_equal(c0.astype(np.int64), ref), ("counts", tag)
        n += 1
    print(f"fuzz ok: {n} cases in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
