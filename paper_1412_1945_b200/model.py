"""Frequency-merged octree background models over a grid of frame regions.

API mirror of the reference's ``octabg.model`` (model.py:1-254).  The bulk
work -- per-(group, region) tree construction and the level-wise frequency
merge -- runs as CUDA kernels in libobg.so (obg_build_presence, obg_merge);
this module validates arguments with the reference's messages, computes the
integer merge cut-off ``k_min`` exactly as the reference's float comparison
would decide it, and keeps results on the device until a host view is asked
for.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from . import _device, _lib
from .errors import FormatError
from .octree import Octree, decode_tree


@dataclass(frozen=True)
class ModelConfig:
    """Training parameters (model.py:20-45)."""

    levels: int = 4
    threshold: float = 0.5
    grid_rows: int = 1
    grid_cols: int = 1
    group_size: int = 1
    training_frames: int = 100

    def __post_init__(self):
        if not 1 <= self.levels <= 8:
            raise ValueError(f"levels must be in 1..8, got {self.levels}")
        if not 0.0 < self.threshold <= 1.0:
            raise ValueError(f"threshold must be in (0, 1], got {self.threshold}")
        if self.grid_rows < 1 or self.grid_cols < 1:
            raise ValueError("grid dimensions must be >= 1")
        if self.group_size < 1:
            raise ValueError("group_size must be >= 1")
        if self.training_frames < self.group_size:
            raise ValueError("training_frames must be >= group_size")


class BackgroundModel:
    """One merged octree per grid region plus the configuration (model.py:48-58).

    Models built on the GPU keep the merged pyramids (``[R*C][PW]`` int32
    words) and the classify operand (leaf cube bitsets, ``[R*C][CW]``) in
    device memory; ``trees`` materialises :class:`Octree` views lazily.
    """

    def __init__(self, config: ModelConfig, frame_width: int, frame_height: int, trees=None, *,
                 _device_pyramids=None, _device_cube=None):
        self.config = config
        self.frame_width = frame_width
        self.frame_height = frame_height
        self._trees = trees
        self._dev_pyr = _device_pyramids
        self._dev_cube = _device_cube
        self._cube_key = None
        if trees is None and _device_pyramids is None:
            raise ValueError("BackgroundModel needs trees")

    @property
    def trees(self) -> list[list[Octree]]:
        if self._trees is None:
            cfg = self.config
            self._trees = [[Octree._from_device(self._dev_pyr[r * cfg.grid_cols + c], cfg.levels)
                            for c in range(cfg.grid_cols)] for r in range(cfg.grid_rows)]
            if self._dev_cube is not None:
                self._cube_key = self._trees_key()
        return self._trees

    def _trees_key(self):
        return tuple((id(t), t._version, t.depth) for row in self._trees for t in row)

    @trees.setter
    def trees(self, value) -> None:
        self._trees = value
        self._dev_pyr = None
        self._dev_cube = None
        self._cube_key = None

    def tree_at(self, row: int, col: int) -> Octree:
        return self.trees[row][col]

    def device_cube(self):
        """Leaf cube bitsets of every region on the device (classify operand)."""
        from . import _device
        cfg = self.config
        if self._dev_cube is not None and self._trees is None:
            return self._dev_cube
        trees = [t for row in self.trees for t in row]
        key = self._trees_key()
        if self._dev_cube is not None and key == self._cube_key:
            return self._dev_cube
        for t in trees:
            if t.depth != cfg.levels:
                raise ValueError(f"tree depth {t.depth} does not match levels {cfg.levels}")
        pyr = _device.torch().stack([t._device() for t in trees])
        cube = _device.empty((len(trees), _lib.cube_words(cfg.levels)), "int32")
        lib = _lib.load()
        _lib.check(lib.obg_leaf_cube(_device.ptr(pyr), len(trees), cfg.levels, _device.ptr(cube),
                                     _device.stream_handle()))
        self._dev_cube, self._cube_key = cube, key
        return cube

    def __eq__(self, other):
        if not isinstance(other, BackgroundModel):
            return NotImplemented
        return (self.config == other.config and self.frame_width == other.frame_width
                and self.frame_height == other.frame_height and self.trees == other.trees)

    def __repr__(self):
        return (f"BackgroundModel(config={self.config!r}, frame_width={self.frame_width}, "
                f"frame_height={self.frame_height})")


def region_of(x: int, y: int, width: int, height: int, grid_rows: int, grid_cols: int) -> tuple[int, int]:
    """Grid cell owning pixel (x, y) (model.py:61-66)."""
    row = min(grid_rows - 1, y * grid_rows // height)
    col = min(grid_cols - 1, x * grid_cols // width)
    return row, col


def region_bounds(extent: int, parts: int) -> list[int]:
    """Slice boundaries b[0..parts]; part p covers [b[p], b[p+1]) (model.py:69-75)."""
    return [(p * extent + parts - 1) // parts for p in range(parts + 1)]


def merge_k_min(total: int, threshold: float) -> int:
    """Smallest k >= 1 with ``k / total >= threshold`` evaluated in IEEE double,
    i.e. exactly the reference's keep test ``len(present) / total >= threshold``
    (model.py:152).  ``ceil(threshold * total)`` is NOT equivalent (e.g. N=100,
    thr=0.55: the reference keeps 55/100 because 0.55 rounds below 55/100)."""
    if total < 1:
        raise ValueError("no trees to merge")
    k = max(1, int(threshold * total) - 1)
    while k > 1 and (k - 1) / total >= threshold:
        k -= 1
    while k / total < threshold:
        k += 1
    return k


def _frames_info(frames):
    """Normalise frames to a sequence/tensor and validate like _check_frames
    (model.py:78-90).  Returns (frames, n, h, w)."""
    from . import _device
    if _device.is_tensor(frames):
        t = _device.torch()
        if frames.ndim == 3:
            frames = frames.unsqueeze(0)
        if frames.ndim != 4 or frames.shape[0] == 0:
            if frames.ndim == 4:
                raise ValueError("no frames given")
            raise ValueError(f"expected (h, w, 3) uint8 frames, got {frames.dtype} {tuple(frames.shape[1:])}")
        if frames.shape[3] != 3 or frames.dtype != t.uint8:
            raise ValueError(f"expected (h, w, 3) uint8 frames, got {frames.dtype} {tuple(frames.shape[1:])}")
        return frames, int(frames.shape[0]), int(frames.shape[1]), int(frames.shape[2])
    if isinstance(frames, np.ndarray) and frames.ndim == 4:
        if frames.shape[0] == 0:
            raise ValueError("no frames given")
        if frames.shape[3] != 3 or frames.dtype != np.uint8:
            raise ValueError(f"expected (h, w, 3) uint8 frames, got {frames.dtype} {frames.shape[1:]}")
        return frames, frames.shape[0], frames.shape[1], frames.shape[2]
    frames = [np.asarray(f) for f in frames]
    if not frames:
        raise ValueError("no frames given")
    first = frames[0]
    if first.ndim != 3 or first.shape[2] != 3 or first.dtype != np.uint8:
        raise ValueError(f"expected (h, w, 3) uint8 frames, got {first.dtype} {first.shape}")
    for i, frame in enumerate(frames):
        if frame.shape != first.shape or frame.dtype != np.uint8:
            raise ValueError(f"frame {i} shape {frame.shape} does not match first frame {first.shape}")
    return frames, len(frames), first.shape[0], first.shape[1]


def _stack_device(frames, n: int):
    """First ``n`` frames as one contiguous (n, h, w, 3) uint8 CUDA tensor."""
    from . import _device
    if _device.is_tensor(frames):
        return _device.to_device_u8(frames[:n])
    if isinstance(frames, np.ndarray):
        return _device.to_device_u8(frames[:n])
    return _device.frames_list_to_device(frames[:n])


def build_presence(frames_dev, levels: int, grid_rows: int = 1, grid_cols: int = 1, group_size: int = 1,
                   counts: bool = False):
    """Batched GPU build: (n, h, w, 3) uint8 CUDA tensor -> per-(group, region)
    pyramids ``[n_groups, R*C, PW]`` (int32 words) and optional per-leaf pixel
    counts ``[n_groups, R*C, 8**L]`` in path-code order."""
    from . import _device
    frames_dev = _device.frames_on_device(frames_dev)
    n, h, w = int(frames_dev.shape[0]), int(frames_dev.shape[1]), int(frames_dev.shape[2])
    n_groups = n // group_size
    n_regions = grid_rows * grid_cols
    lib = _lib.load()
    pw = _lib.pyramid_words(levels)
    out = _device.empty((n_groups, n_regions, pw), "int32")
    cnt = _device.empty((n_groups, n_regions, 8 ** levels), "int32") if counts else None
    ws_bytes = lib.obg_build_workspace_bytes(n_groups, n_regions, levels)
    stream = _device.stream_handle()
    ws = _workspace(ws_bytes, stream)
    try:
        _lib.check(lib.obg_build_presence(
            _device.ptr(frames_dev), n, h, w, levels, grid_rows, grid_cols, group_size, _device.ptr(out),
            _device.ptr(cnt) if cnt is not None else None, _device.ptr(ws), ws_bytes, _lib.WS_ZEROED, stream))
    except Exception:
        _drop_workspace(stream)
        raise
    return (out, cnt) if counts else out


# Build workspaces kept per (device, stream): obg_build_presence hands its
# workspace back all-zero, so a kept one skips the clearing memset.  Keyed
# strictly by stream because concurrent builds must not share one.  Only eager
# calls use this cache: a CUDA graph holds its workspace's pointer for every
# replay, so captures get a workspace of their own (passed in explicitly, as
# pipeline.CapturedStep does, or allocated here and kept alive for the
# process) -- never one that the cache could replace or drop.
_WORKSPACES: dict = {}
_CAPTURE_WORKSPACES: list = []


def new_workspace(nbytes: int):
    """A zeroed build workspace of ``nbytes`` (owned by the caller)."""
    t = _device.torch()
    return t.zeros((max(nbytes, 4) + 3) // 4, dtype=t.int32, device="cuda")


def _workspace(nbytes: int, stream: int, explicit=None):
    t = _device.torch()
    if explicit is not None:
        if explicit.numel() * 4 < nbytes or not explicit.is_cuda:
            raise ValueError(f"workspace must be a CUDA tensor of >= {nbytes} bytes")
        return explicit
    if t.cuda.is_current_stream_capturing():
        ws = new_workspace(nbytes)      # zeroed once at capture; zero-on-return keeps it so
        _CAPTURE_WORKSPACES.append(ws)
        return ws
    key = (t.cuda.current_device(), stream)
    ws = _WORKSPACES.get(key)
    if ws is None or ws.numel() * 4 < nbytes:
        ws = new_workspace(nbytes)
        _WORKSPACES[key] = ws
    return ws


def _drop_workspace(stream: int, explicit=None) -> None:
    """After a failed launch the workspace state is unknown: drop a cached
    eager one (an explicit one is re-zeroed)."""
    t = _device.torch()
    if explicit is not None:
        explicit.zero_()
    elif not t.cuda.is_current_stream_capturing():
        _WORKSPACES.pop((t.cuda.current_device(), stream), None)


def merge_pyramids(pyramids_dev, levels: int, k_min: int, with_cube: bool = False):
    """GPU merge: ``[n_trees, R*C, PW]`` -> merged ``[R*C, PW]`` (and, with
    ``with_cube``, the merged leaves in cube order ``[R*C, CW]`` for classify)."""
    from . import _device
    n_trees, n_regions = int(pyramids_dev.shape[0]), int(pyramids_dev.shape[1])
    out = _device.empty((n_regions, _lib.pyramid_words(levels)), "int32")
    cube = _device.empty((n_regions, _lib.cube_words(levels)), "int32") if with_cube else None
    lib = _lib.load()
    _lib.check(lib.obg_merge(_device.ptr(pyramids_dev), n_trees, n_regions, levels, k_min, _device.ptr(out),
                             _device.ptr(cube) if with_cube else None, _device.stream_handle()))
    return (out, cube) if with_cube else out


def build_frame_tree(frames, region: tuple[int, int], config: ModelConfig) -> Octree:
    """Tree of every quantized colour seen in ``region`` across one frame group
    (model.py:93-109), built by obg_build_presence on the region's block."""
    frames = [np.asarray(f) for f in frames]
    if len(frames) != config.group_size:
        raise ValueError(f"expected a group of {config.group_size} frames, got {len(frames)}")
    _, _, h, w = _frames_info(frames)
    row, col = region
    if not (0 <= row < config.grid_rows and 0 <= col < config.grid_cols):
        raise ValueError(f"region {region} outside {config.grid_rows}x{config.grid_cols} grid")
    rows = region_bounds(h, config.grid_rows)
    cols = region_bounds(w, config.grid_cols)
    from . import _device
    if (rows[row], rows[row + 1], cols[col], cols[col + 1]) == (0, h, 0, w) and h * w > 0:
        # the region is the whole frame (1x1 grids): no block copy, the frames
        # go up through pinned staging (pool gather + asynchronous H2D)
        _device.require_cuda()
        dev = _device.frames_list_to_device(frames)
    else:
        blocks = np.stack([f[rows[row]:rows[row + 1], cols[col]:cols[col + 1]] for f in frames])
        if blocks.shape[1] == 0 or blocks.shape[2] == 0:
            return Octree(config.levels)
        _device.require_cuda()
        dev = _device.to_device_u8(blocks)
    pyr = build_presence(dev, config.levels, 1, 1, len(frames))
    return Octree._from_device(pyr[0, 0], config.levels)


def merge_trees(trees, threshold: float, levels: int) -> Octree:
    """Level-wise frequency merge (model.py:112-154) on the GPU.

    A node survives iff the number of input trees holding it is >= k_min,
    with k_min the smallest count whose fraction of *all* input trees (empty
    ones included) passes the reference's float test.  Because input trees are
    parent-closed, this per-level rule reproduces the reference's top-down
    recursion exactly, dead-end branches included."""
    trees = list(trees)
    if not trees:
        raise ValueError("no trees to merge")
    if not 0.0 < threshold <= 1.0:
        raise ValueError(f"threshold must be in (0, 1], got {threshold}")
    for tree in trees:
        if tree.depth != levels:
            raise ValueError(f"tree depth {tree.depth} does not match levels {levels}")
    from . import _device
    _device.require_cuda()
    k_min = merge_k_min(len(trees), threshold)
    pyr = _device.torch().stack([t._device() for t in trees]).unsqueeze(1)
    merged = merge_pyramids(pyr.contiguous(), levels, k_min)
    return Octree._from_device(merged[0], levels)


def build_background_model(frames, config: ModelConfig) -> BackgroundModel:
    """Train a model from the first ``config.training_frames`` frames
    (model.py:157-185): one GPU build over every group x region, one GPU merge
    per region, and the classify operand prepared on the device."""
    frames, n, h, w = _frames_info(frames)
    usable = min(n, config.training_frames)
    n_groups = usable // config.group_size
    if n_groups == 0:
        raise ValueError(f"need at least {config.group_size} frames for one group, got {usable}")
    from . import _device
    _device.require_cuda()
    dev = _stack_device(frames, n_groups * config.group_size)
    return build_background_model_device(dev, config, n_groups=n_groups)


def build_background_model_device(frames_dev, config: ModelConfig, n_groups: int | None = None,
                                  workspace=None) -> BackgroundModel:
    """Same as :func:`build_background_model` for a CUDA (n, h, w, 3) uint8
    tensor that already holds the training frames (no host round trip).
    ``workspace``: a caller-owned zeroed buffer (``new_workspace``) of at
    least ``obg_build_workspace_bytes`` -- what a captured graph should use."""
    from . import _device
    frames_dev = _device.frames_on_device(frames_dev)
    n, h, w = int(frames_dev.shape[0]), int(frames_dev.shape[1]), int(frames_dev.shape[2])
    if n_groups is None:
        n_groups = min(n, config.training_frames) // config.group_size
        if n_groups == 0:
            raise ValueError(f"need at least {config.group_size} frames for one group, got {n}")
        frames_dev = frames_dev[: n_groups * config.group_size]
    L, R, C, gs = config.levels, config.grid_rows, config.grid_cols, config.group_size
    n_regions = R * C
    lib = _lib.load()
    pw = _lib.pyramid_words(L)
    trees = _device.empty((n_groups, n_regions, pw), "int32")
    merged = _device.empty((n_regions, pw), "int32")
    cube = _device.empty((n_regions, _lib.cube_words(L)), "int32")
    ws_bytes = lib.obg_build_workspace_bytes(n_groups, n_regions, L)
    stream = _device.stream_handle()
    ws = _workspace(ws_bytes, stream, workspace)
    try:
        _lib.check(lib.obg_build_model(
            _device.ptr(frames_dev), n_groups * gs, h, w, L, R, C, gs, merge_k_min(n_groups, config.threshold),
            _device.ptr(trees), _device.ptr(merged), _device.ptr(cube), _device.ptr(ws), ws_bytes, _lib.WS_ZEROED,
            stream))
    except Exception:
        _drop_workspace(stream, workspace)
        raise
    return BackgroundModel(config, frame_width=w, frame_height=h, _device_pyramids=merged, _device_cube=cube)


# ---------------------------------------------------------------------------
# OBGM model file (model.py:188-254): magic, version, levels, grid, frame size,
# threshold x10000, then row-major region records (presence byte + preorder
# tree bytes).
# ---------------------------------------------------------------------------
_MAGIC = b"OBGM"
_VERSION = 1
_HEADER = struct.Struct("<4sBBHHIIH")


def write_model(model: BackgroundModel) -> bytes:
    cfg = model.config
    out = bytearray(_HEADER.pack(_MAGIC, _VERSION, cfg.levels, cfg.grid_rows, cfg.grid_cols,
                                 model.frame_width, model.frame_height, round(cfg.threshold * 10000)))
    for row in model.trees:
        for tree in row:
            if tree.is_empty:
                out.append(0)
            else:
                out.append(1)
                out += tree.to_bytes()
    return bytes(out)


def read_model(data: bytes) -> BackgroundModel:
    if len(data) < _HEADER.size:
        raise FormatError("truncated model header", len(data))
    magic, version, levels, rows, cols, width, height, thr_fp = _HEADER.unpack_from(data)
    if magic != _MAGIC:
        raise FormatError(f"bad magic {magic!r}, expected {_MAGIC!r}", 0)
    if version != _VERSION:
        raise FormatError(f"unsupported model version {version}", 4)
    config = ModelConfig(levels=levels, threshold=thr_fp / 10000.0, grid_rows=rows, grid_cols=cols,
                         group_size=1, training_frames=1)
    pos = _HEADER.size
    trees: list[list[Octree]] = []
    for _ in range(rows):
        tree_row = []
        for _ in range(cols):
            if pos >= len(data):
                raise FormatError("truncated region record", pos)
            flag = data[pos]
            pos += 1
            if flag == 0:
                tree_row.append(Octree(levels))
            elif flag == 1:
                tree, pos = decode_tree(data, pos, levels)
                tree_row.append(tree)
            else:
                raise FormatError(f"bad region presence flag {flag}", pos - 1)
        trees.append(tree_row)
    if pos != len(data):
        raise FormatError("trailing data after model", pos)
    return BackgroundModel(config, frame_width=width, frame_height=height, trees=trees)


def save_model(path, model: BackgroundModel) -> None:
    with open(path, "wb") as f:
        f.write(write_model(model))


def load_model(path) -> BackgroundModel:
    with open(path, "rb") as f:
        return read_model(f.read())
