"""Shared test helpers (digests, oracle adaptors)."""

from __future__ import annotations

import hashlib

import numpy as np

from oracle import octree_oracle as orc


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


def mask_digest(mask: np.ndarray) -> str:
    return sha(np.packbits(np.asarray(mask).astype(bool).ravel(), bitorder="little"))


def mask_hex(mask: np.ndarray) -> str:
    return np.packbits(np.asarray(mask).astype(bool).ravel(), bitorder="little").tobytes().hex()


def oracle_group_trees(frames, levels, rows, cols, gs):
    n_groups = len(frames) // gs
    return [[[orc.build_frame_tree(frames[g * gs:(g + 1) * gs], (r, c), levels, rows, cols)
              for c in range(cols)] for r in range(rows)] for g in range(n_groups)]
