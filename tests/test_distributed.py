"""Sharded training (paper_1412_1945_b200.distributed) on CPU with gloo,
world_size 2: the count all-reduce + global k_min reproduce the reference's
merge over the concatenated shards."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1412_1945_b200 import Octree, _lib, merge_k_min
from paper_1412_1945_b200.distributed import allreduce_counts


def _pyramid(tree, levels):
    from oracle import octree_oracle as orc
    blob = orc.to_bytes(tree)
    return (Octree.from_bytes(blob, levels) if blob else Octree(levels))._host()


def _counts(trees, levels):
    bits = np.stack([np.unpackbits(_pyramid(t, levels).view(np.uint8), bitorder="little") for t in trees])
    return bits.sum(axis=0).astype(np.int32)[None, :]          # [R=1, PW*32]


def _threshold(counts, k_min):
    c = counts.reshape(counts.shape[0], -1, 32) >= k_min
    return np.packbits(c, axis=2, bitorder="little").view(np.uint32)[..., 0]


def _worker(rank, world, port, frames, levels, threshold, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import octree_oracle as orc
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shard = frames[rank::world]
    trees = [orc.build_frame_tree([f], (0, 0), levels, 1, 1) for f in shard]
    counts = torch.from_numpy(_counts(trees, levels))
    total = allreduce_counts(counts, len(trees))
    merged = _threshold(counts.numpy(), merge_k_min(total, threshold))
    q.put((rank, total, merged))
    dist.destroy_process_group()


@pytest.mark.parametrize("levels,threshold", [(3, 0.5), (4, 0.3), (2, 0.55)])
def test_sharded_merge_equals_global_merge(levels, threshold):
    from oracle import octree_oracle as orc
    rng = np.random.default_rng(levels)
    base = rng.integers(0, 256, size=(1, 1, 1, 3))
    frames = np.clip(base + rng.integers(-60, 61, size=(9, 10, 12, 3)), 0, 255).astype(np.uint8)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + levels * 7 + int(threshold * 100)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, frames, levels, threshold, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_tree = orc.build_background_model(list(frames), levels, threshold)[(0, 0)]
    want = _pyramid(want_tree, levels)
    for rank, total, merged in results:
        assert total == len(frames)
        assert np.array_equal(merged[0], want), rank


def test_single_process_is_identity():
    c = torch.arange(64, dtype=torch.int32)
    assert allreduce_counts(c, 5) == 5
    assert torch.equal(c, torch.arange(64, dtype=torch.int32))
    assert _lib.pyramid_words(3) == 19
