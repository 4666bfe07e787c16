"""CPU ORACLE -- test infrastructure only, never part of the product path.

A numpy restatement of the reference's octree background-model path
(/root/reference/pkg/src/octabg), used by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg as the checker.  It is pinned against golden
vectors produced by the reference itself (tests/golden/make_golden.py) in
tests/test_oracle.py.  Nothing under paper_1412_1945_b200/ may import it.

A tree is represented as ``OracleTree(depth, root, levels)`` where
``levels[l]`` (l = 1..depth) is the sorted array of level-l node codes (the
l-digit path prefixes).  This is the node set of the reference's pointer
tree, so ``to_bytes`` can be compared byte for byte.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


# --- octree.py:21-35  spread tables ------------------------------------------
def _spread_table(offset: int) -> np.ndarray:
    table = np.zeros(256, dtype=np.uint32)
    for value in range(256):
        s = 0
        for i in range(8):
            s |= ((value >> i) & 1) << (3 * i + offset)
        table[value] = s
    return table


SPREAD_R = _spread_table(2)
SPREAD_G = _spread_table(1)
SPREAD_B = _spread_table(0)


# --- octree.py:83-90  pack_codes ------------------------------------------------
def pack_codes(pixels: np.ndarray, levels: int) -> np.ndarray:
    pixels = np.asarray(pixels)
    assert pixels.dtype == np.uint8 and pixels.shape[-1] == 3
    codes = SPREAD_R[pixels[..., 0]] | SPREAD_G[pixels[..., 1]] | SPREAD_B[pixels[..., 2]]
    return codes >> np.uint32(3 * (8 - levels))


# --- model.py:69-75  region_bounds ------------------------------------------------
def region_bounds(extent: int, parts: int) -> list[int]:
    return [(p * extent + parts - 1) // parts for p in range(parts + 1)]


@dataclass
class OracleTree:
    depth: int
    root: bool = False
    levels: dict = field(default_factory=dict)   # l -> sorted unique int64 codes

    def level(self, l: int) -> np.ndarray:
        return self.levels.get(l, np.zeros(0, dtype=np.int64))

    def leaf_codes(self) -> list[int]:
        # octree.py:206-211 / 293-300: full-depth leaves ascending
        return self.level(self.depth).tolist() if self.root else []

    def node_count(self) -> int:
        return (1 + sum(len(self.level(l)) for l in range(1, self.depth + 1))) if self.root else 0


# --- octree.py:158-169 store_code, applied to a set of codes -------------------------
def tree_from_codes(codes, depth: int) -> OracleTree:
    codes = np.unique(np.asarray(codes, dtype=np.int64))
    t = OracleTree(depth, root=codes.size > 0)
    for l in range(1, depth + 1):
        t.levels[l] = np.unique(codes >> (3 * (depth - l)))
    return t


# --- model.py:93-109  build_frame_tree -------------------------------------------------
def build_frame_tree(frames, region, levels, grid_rows, grid_cols) -> OracleTree:
    h, w = frames[0].shape[:2]
    rows, cols = region_bounds(h, grid_rows), region_bounds(w, grid_cols)
    r, c = region
    codes = [np.unique(pack_codes(f[rows[r]:rows[r + 1], cols[c]:cols[c + 1]], levels)) for f in frames]
    codes = np.unique(np.concatenate(codes)) if codes else np.zeros(0, dtype=np.int64)
    return tree_from_codes(codes, levels)


# --- model.py:112-154  merge_trees, closed form ---------------------------------------
def merge_trees(trees: list[OracleTree], threshold: float, levels: int) -> OracleTree:
    """Level-wise keep iff (#trees holding the node) / total >= threshold, as
    the reference compares (float division, model.py:152).  Input trees are
    parent-closed, so the top-down recursion equals this per-level rule;
    merge_trees_recursive below restates the recursion for small cases."""
    total = len(trees)
    out = OracleTree(levels)
    for l in range(1, levels + 1):
        arrs = [t.level(l) for t in trees if t.root]
        if not arrs:
            out.levels[l] = np.zeros(0, dtype=np.int64)
            continue
        vals, counts = np.unique(np.concatenate(arrs), return_counts=True)
        out.levels[l] = vals[counts / total >= threshold].astype(np.int64)
    out.root = len(out.level(1)) > 0
    if not out.root:
        out.levels = {}
    return out


def merge_trees_recursive(trees: list[OracleTree], threshold: float, levels: int) -> OracleTree:
    """Direct restatement of _merge_nodes (model.py:140-154) on node sets."""
    total = len(trees)
    sets = [[set(t.level(l).tolist()) for l in range(levels + 1)] for t in trees if t.root]
    kept = {l: [] for l in range(1, levels + 1)}

    def rec(present, prefix, level):
        if level == levels:
            return
        for k in range(8):
            child = prefix * 8 + k
            have = [s for s in present if child in s[level + 1]]
            if have and len(have) / total >= threshold:
                kept[level + 1].append(child)
                rec(have, child, level + 1)

    if sets:
        rec(sets, 0, 0)
    out = OracleTree(levels, root=bool(kept[1]))
    if out.root:
        out.levels = {l: np.array(sorted(v), dtype=np.int64) for l, v in kept.items()}
    return out


# --- octree.py:217-227, 258-267  to_bytes (preorder child masks) ------------------------
def to_bytes(tree: OracleTree) -> bytes:
    if not tree.root:
        return b""
    L = tree.depth
    nodes = [(0, np.array([0], dtype=np.int64))] + [(l, tree.level(l)) for l in range(1, L + 1)]
    all_key, all_lev, all_mask = [], [], []
    for l, codes in nodes:
        if codes.size == 0:
            continue
        if l < L:
            child = tree.level(l + 1)
            parent_of_child = child >> 3
            m = np.zeros(codes.size, dtype=np.int64)
            idx = np.searchsorted(codes, parent_of_child)
            np.bitwise_or.at(m, idx, np.left_shift(1, child & 7))
        else:
            m = np.zeros(codes.size, dtype=np.int64)
        all_key.append(codes << (3 * (L - l)))
        all_lev.append(np.full(codes.size, l))
        all_mask.append(m)
    key = np.concatenate(all_key)
    lv = np.concatenate(all_lev)
    mk = np.concatenate(all_mask)
    order = np.lexsort((lv, key))          # preorder: by padded path, ancestors first
    return mk[order].astype(np.uint8).tobytes()


# --- model.py:157-185  build_background_model -------------------------------------------
def build_background_model(frames, levels, threshold, grid_rows=1, grid_cols=1, group_size=1,
                           training_frames=None):
    usable = frames if training_frames is None else frames[:training_frames]
    n_groups = len(usable) // group_size
    assert n_groups >= 1
    trees = {}
    for r in range(grid_rows):
        for c in range(grid_cols):
            group_trees = [build_frame_tree(usable[g * group_size:(g + 1) * group_size], (r, c), levels,
                                            grid_rows, grid_cols) for g in range(n_groups)]
            trees[(r, c)] = merge_trees(group_trees, threshold, levels)
    return trees


# --- detect.py:22-53  detect_octree -------------------------------------------------------
def detect_octree(trees, frame, levels, grid_rows=1, grid_cols=1) -> np.ndarray:
    codes = pack_codes(frame, levels)
    h, w = frame.shape[:2]
    rows, cols = region_bounds(h, grid_rows), region_bounds(w, grid_cols)
    fg = np.zeros(codes.shape, dtype=bool)
    for r in range(grid_rows):
        for c in range(grid_cols):
            block = codes[rows[r]:rows[r + 1], cols[c]:cols[c + 1]]
            if block.size == 0:
                continue
            leaves = trees[(r, c)].leaf_codes()
            if leaves:
                bg = np.isin(block, np.asarray(leaves, dtype=codes.dtype))
            else:
                bg = np.zeros(block.shape, dtype=bool)
            fg[rows[r]:rows[r + 1], cols[c]:cols[c + 1]] = ~bg
    return fg


# --- superset the reference does not compute: per-leaf occupancy counts ---------------
def leaf_counts(frames, levels) -> np.ndarray:
    """np.bincount(pack_codes(...)) over a frame group."""
    codes = np.concatenate([pack_codes(f, levels).ravel() for f in frames])
    return np.bincount(codes, minlength=8 ** levels).astype(np.int64)


def prune(tree: OracleTree, new_depth: int) -> OracleTree:
    """octree.py:193-204: keep levels 1..new_depth."""
    out = OracleTree(new_depth, root=tree.root)
    out.levels = {l: tree.level(l) for l in range(1, new_depth + 1)} if tree.root else {}
    return out


# --- evaluation.py:38-53 (accumulate): confusion counts, foreground positive ----------
def confusion(predicted, truth) -> tuple:
    """(tn, tp, fn, fp) of one predicted / truth mask pair (evaluation.py:38-53)."""
    p = np.asarray(predicted, dtype=bool)
    t = np.asarray(truth, dtype=bool)
    if p.shape != t.shape:
        raise ValueError(f"mask dimensions {p.shape} vs {t.shape} do not match")
    return (int(np.count_nonzero(~p & ~t)), int(np.count_nonzero(p & t)),
            int(np.count_nonzero(~p & t)), int(np.count_nonzero(p & ~t)))


# --- detect.py:56-63  detect_frame_diff (comparison baseline) --------------------------
def detect_frame_diff(previous, current, diff_threshold: int = 30) -> np.ndarray:
    previous = np.asarray(previous)
    current = np.asarray(current)
    assert previous.shape[:2] == current.shape[:2]
    delta = np.abs(current.astype(np.int16) - previous.astype(np.int16)).max(axis=2)
    return delta > diff_threshold


# --- detect.py:66-83  detect_running_average (comparison baseline) ---------------------
def detect_running_average(frames_seen: int, average, current, diff_threshold: int = 30):
    average = np.asarray(average, dtype=np.float64)
    current = np.asarray(current)
    assert average.shape[:2] == current.shape[:2]
    delta = np.abs(current.astype(np.float64) - average).max(axis=2)
    mask = delta > diff_threshold
    updated = average + (current - average) / (frames_seen + 1)
    return mask, updated
