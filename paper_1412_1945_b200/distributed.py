"""Multi-GPU training of one background model.

Training frames are independent units: each rank builds the per-(group,
region) trees of its own shard and counts, per node, how many of its trees
hold it (obg_build_counts).  The only exchange is one
all-reduce(SUM) of those counts plus the tree total; every rank then applies
the reference's threshold locally (obg_merge_threshold), so all ranks end up
with the identical merged model -- the one the reference would build from the
concatenation of the shards (obg_threshold_counts) (merge_trees is permutation invariant,
reference tests/test_model.py:154-161).

Classification needs no communication: each rank classifies its own frames
against its replica of the (small) merged model.
"""

from __future__ import annotations

from . import _device, _lib
from .model import BackgroundModel, ModelConfig, merge_k_min


def allreduce_counts(counts, n_trees: int, group=None):
    """Sum per-node tree counts and the tree total over the process group.

    ``counts`` is modified in place; returns the global tree total.  Works on
    CUDA tensors (NCCL) and CPU tensors (gloo)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return n_trees
    total = torch.tensor([n_trees], dtype=torch.int64, device=counts.device)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(total, op=dist.ReduceOp.SUM, group=group)
    return int(total.item())


def build_background_model_sharded(frames_dev, config: ModelConfig, group=None, global_trees: int | None = None):
    """Build the model from this rank's CUDA frame shard (n, h, w, 3) uint8.

    Every rank's shard must hold whole groups (its length is floored to a
    multiple of ``group_size``).  ``global_trees`` (the total number of trees
    over all ranks) may be passed to skip the scalar all-reduce; ``k_min`` is
    computed from it exactly as the reference's float test (model.py:152).

    Device path: ``obg_build_counts`` (the cube-order build of
    ``obg_build_model`` with per-node tree counts instead of its threshold),
    one all-reduce(SUM) of the counts, ``obg_threshold_counts`` (threshold +
    path-order conversion + classify operand)."""
    from .model import _drop_workspace, _workspace
    frames_dev = _device.frames_on_device(frames_dev)
    n, h, w = int(frames_dev.shape[0]), int(frames_dev.shape[1]), int(frames_dev.shape[2])
    n_groups = n // config.group_size
    if n_groups == 0:
        raise ValueError(f"need at least {config.group_size} frames for one group, got {n}")
    L = config.levels
    R, C, gs = config.grid_rows, config.grid_cols, config.group_size
    n_regions = R * C
    lib = _lib.load()
    pw = _lib.pyramid_words(L)
    frames_dev = _device.to_device_u8(frames_dev[: n_groups * gs])
    counts = _device.empty((n_regions, pw * 32), "int32")
    ws_bytes = lib.obg_build_workspace_bytes(n_groups, n_regions, L)
    stream = _device.stream_handle()
    ws = _workspace(ws_bytes, stream)
    try:
        _lib.check(lib.obg_build_counts(_device.ptr(frames_dev), n_groups * gs, h, w, L, R, C, gs,
                                        _device.ptr(counts), _device.ptr(ws), ws_bytes, _lib.WS_ZEROED, stream))
    except Exception:
        _drop_workspace(stream)
        raise
    if global_trees is None:
        total = allreduce_counts(counts, n_groups, group)
    else:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
        total = global_trees
    k_min = merge_k_min(total, config.threshold)
    merged = _device.empty((n_regions, pw), "int32")
    cube = _device.empty((n_regions, _lib.cube_words(L)), "int32")
    _lib.check(lib.obg_threshold_counts(_device.ptr(counts), n_regions, L, k_min, _device.ptr(merged),
                                        _device.ptr(cube), stream))
    return BackgroundModel(config, frame_width=w, frame_height=h, _device_pyramids=merged, _device_cube=cube)
