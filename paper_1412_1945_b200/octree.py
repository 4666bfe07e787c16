"""Fixed-depth presence octrees over 8-bit RGB, stored as per-level bitsets.

API mirror of the reference's ``octabg.octree`` (octree.py:1-300).  The
reference keeps a pointer tree of ``_Node`` objects; here a tree of depth L is
its *pyramid*: for every level l = 1..L a bitset of 8**l bits in path-code
order (bit c set <=> the node whose path is the l octal digits of c exists),
plus a root flag.  Because a tree's node set is closed under "parent of", the
pyramid is an exact, canonical representation of every reference tree,
including merged trees with dead-end interior nodes (model.py:119-120) and
root-only trees from ``from_bytes(b"\\x00")``.

The child-mask byte the reference serialises for node p at level l
(octree.py:258-267) is simply byte p of level l+1, so ``to_bytes`` is a
rank computation instead of a recursive walk.

Trees produced by the GPU path (build / merge) keep their pyramid in device
memory and are copied to the host only when a host method needs it.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import FormatError

Color = tuple[int, int, int]


def _spread_table(offset: int) -> np.ndarray:
    """Channel bit i -> bit 3i+offset (reference _spread_table, octree.py:21-29)."""
    v = np.arange(256, dtype=np.uint32)
    out = np.zeros(256, dtype=np.uint32)
    for i in range(8):
        out |= ((v >> np.uint32(i)) & np.uint32(1)) << np.uint32(3 * i + offset)
    return out


_SPREAD = (_spread_table(2), _spread_table(1), _spread_table(0))


def _check_levels(levels: int) -> None:
    if not 1 <= levels <= 8:
        raise ValueError(f"levels must be in 1..8, got {levels}")


def _check_color(color: Color) -> None:
    r, g, b = color
    if not (0 <= r <= 255 and 0 <= g <= 255 and 0 <= b <= 255):
        raise ValueError(f"color channels must be in 0..255, got {color}")


def child_index(color: Color, bit_position: int) -> int:
    """Child slot (0..7) selected by one bit plane; 7 is the MSB (octree.py:49-56)."""
    r, g, b = color
    return (((r >> bit_position) & 1) << 2) | (((g >> bit_position) & 1) << 1) | ((b >> bit_position) & 1)


def quantize_color(color: Color, levels: int) -> Color:
    """Keep the top ``levels`` bits per channel (octree.py:59-67)."""
    _check_levels(levels)
    mask = (0xFF << (8 - levels)) & 0xFF
    r, g, b = color
    return (r & mask, g & mask, b & mask)


def pack_code(color: Color, levels: int) -> int:
    """Root-to-leaf path as ``levels`` octal digits (octree.py:70-80)."""
    _check_levels(levels)
    _check_color(color)
    r, g, b = color
    code = int(_SPREAD[0][r] | _SPREAD[1][g] | _SPREAD[2][b])
    return code >> (3 * (8 - levels))


def pack_codes(pixels, levels: int) -> np.ndarray:
    """Path code of every pixel of an ``(..., 3)`` uint8 array (octree.py:83-90).

    Computed on the GPU by ``obg_pack_codes``; returns a host uint32 array of
    shape ``pixels.shape[:-1]`` (a CUDA tensor in, a CUDA tensor out).
    """
    _check_levels(levels)
    from . import _device
    if _device.is_tensor(pixels):
        t = _device.torch()
        if pixels.shape[-1] != 3 or pixels.dtype != t.uint8:
            raise ValueError(f"expected (..., 3) uint8 pixels, got {pixels.dtype} {tuple(pixels.shape)}")
        shape, as_tensor = tuple(pixels.shape[:-1]), True
        dev = _device.to_device_u8(pixels)
    else:
        pixels = np.asarray(pixels)
        if pixels.shape[-1] != 3 or pixels.dtype != np.uint8:
            raise ValueError(f"expected (..., 3) uint8 pixels, got {pixels.dtype} {pixels.shape}")
        shape, as_tensor = pixels.shape[:-1], False
        if pixels.size == 0:
            return np.zeros(shape, dtype=np.uint32)
        _device.require_cuda()
        dev = _device.to_device_u8(pixels)
    n = int(np.prod(shape)) if shape else 1
    out = _device.empty((max(n, 1),), "int32")
    lib = _lib.load()
    _lib.check(lib.obg_pack_codes(_device.ptr(dev), n, levels, _device.ptr(out), _device.stream_handle()))
    out = out[:n].reshape(shape)
    if as_tensor:
        return out
    return _device.u32_to_numpy(out).reshape(shape)


def code_to_color(code: int, levels: int) -> Color:
    """Zero-filled representative colour of a path code (octree.py:93-103)."""
    _check_levels(levels)
    r = g = b = 0
    for k in range(levels):
        digit = (code >> (3 * (levels - 1 - k))) & 7
        bit = 7 - k
        r |= ((digit >> 2) & 1) << bit
        g |= ((digit >> 1) & 1) << bit
        b |= (digit & 1) << bit
    return (r, g, b)


# ---------------------------------------------------------------------------
# level helpers (host side)
# ---------------------------------------------------------------------------
_EMPTY = np.zeros(0, dtype=np.int64)
_EMPTY.flags.writeable = False


def _level_bits(pyr: np.ndarray, level: int) -> np.ndarray:
    """Level ``level`` of a dense pyramid as a bool array of 8**level entries."""
    off, nw = _lib.level_offset(level), _lib.level_words(level)
    bits = np.unpackbits(pyr[off:off + nw].view(np.uint8), bitorder="little")
    return bits[: 8 ** level].astype(bool)


def _level_codes(pyr: np.ndarray, level: int) -> np.ndarray:
    """Ascending codes of the set bits of one dense pyramid level; only the
    non-zero words are expanded, so a sparse depth-8 level costs O(words)."""
    off, nw = _lib.level_offset(level), _lib.level_words(level)
    words = pyr[off:off + nw]
    nz = np.flatnonzero(words)
    if nz.size == 0:
        return _EMPTY
    bits = np.unpackbits(words[nz].view(np.uint8), bitorder="little").reshape(-1, 32)
    row, col = np.nonzero(bits)
    return nz[row].astype(np.int64) * 32 + col


def _codes_to_words(codes: np.ndarray, level: int) -> np.ndarray:
    """Dense u32 words of one level from its codes."""
    nw = _lib.level_words(level)
    if codes.size * 16 < nw * 32:
        words = np.zeros(nw, dtype=np.uint32)
        np.bitwise_or.at(words, codes >> 5, np.left_shift(np.uint32(1), (codes & 31).astype(np.uint32)))
        return words
    bits = np.zeros(nw * 32, dtype=bool)
    bits[codes] = True
    return np.packbits(bits, bitorder="little").view(np.uint32)


def _child_masks(parents: np.ndarray, children: np.ndarray) -> np.ndarray:
    """Child-mask byte of every node in ``parents`` (ascending codes of level
    l) from the ascending codes of level l+1: bit k <=> child 8p+k present."""
    out = np.zeros(parents.size, dtype=np.uint8)
    if children.size:
        idx = np.searchsorted(parents, children >> 3)
        out[:] = np.bincount(idx, weights=np.left_shift(1, children & 7), minlength=parents.size)
    return out


class _NodeView:
    """Read-only stand-in for the reference's ``_Node`` (octree.py:106-110):
    ``children`` is the list of 8 child views (None where absent)."""

    __slots__ = ("_tree", "_level", "_prefix")

    def __init__(self, tree: "Octree", level: int, prefix: int):
        self._tree, self._level, self._prefix = tree, level, prefix

    @property
    def children(self) -> list:
        t = self._tree
        if self._level >= t.depth:
            return [None] * 8
        kids = t._levels()[self._level + 1]
        lo, hi = np.searchsorted(kids, [self._prefix * 8, self._prefix * 8 + 8])
        present = {int(c) & 7 for c in kids[lo:hi]}
        return [_NodeView(t, self._level + 1, self._prefix * 8 + k) if k in present else None for k in range(8)]


class Octree:
    """Presence tree over quantized colours, leaves at a fixed depth (octree.py:113-247).

    The node set of a tree is closed under "parent of", so a tree is exactly
    its root flag plus, per level l = 1..depth, the set of l-digit path codes
    present.  That set is held in whichever of three forms the last producer
    left, converted on demand:

    * host, sparse: one ascending int64 code array per level (O(nodes); what
      ``store``/``from_bytes``/host reads use),
    * host, dense: the u32 pyramid (8**l bits per level, path-code order),
    * device: the same pyramid as a CUDA int32 tensor (GPU build / merge
      output, classify operand source).

    ``to_bytes`` of a device-resident tree runs on the GPU (``obg_serialize``);
    a tree decoded by ``from_bytes`` keeps its bytes (the encoding is a
    bijection, so re-encoding an unmodified tree reproduces them).
    """

    __slots__ = ("depth", "_lv", "_pend", "_pyr", "_dev", "_bytes", "_has_root", "_version")

    def __init__(self, depth: int):
        _check_levels(depth)
        self.depth = depth
        self._lv: list | None = [None] + [_EMPTY] * depth   # sparse form (index = level)
        self._pend: list = []             # leaf codes stored since the last normalisation
        self._pyr: np.ndarray | None = None   # dense host pyramid (u32 words)
        self._dev = None                  # CUDA pyramid (int32 words)
        self._bytes: bytes | None = None  # cached preorder serialisation
        self._has_root: bool | None = False   # None: level 1 non-empty (device trees)
        self._version = 0

    # -- construction ---------------------------------------------------------
    @classmethod
    def _from_pyramid(cls, pyramid: np.ndarray, depth: int, has_root: bool | None = None) -> "Octree":
        tree = cls(depth)
        pyr = np.ascontiguousarray(pyramid, dtype=np.uint32).copy()
        if len(pyr) != _lib.pyramid_words(depth):
            raise ValueError("pyramid size does not match depth")
        tree._lv, tree._pyr = None, pyr
        tree._has_root = bool(pyr[0] & 0xFF) if has_root is None else bool(has_root)
        return tree

    @classmethod
    def _from_levels(cls, levels: list, depth: int, has_root: bool) -> "Octree":
        tree = cls(depth)
        tree._lv = [None] + [np.asarray(c, dtype=np.int64) for c in levels[1:depth + 1]]
        tree._has_root = bool(has_root)
        return tree

    @classmethod
    def _from_device(cls, dev_pyramid, depth: int) -> "Octree":
        """Tree backed by a CUDA pyramid (GPU build/merge output).  Its root
        exists iff level 1 is non-empty, which holds for built trees
        (model.py:93-109) and merged trees (model.py:133-136)."""
        tree = cls(depth)
        tree._lv = None
        tree._dev = dev_pyramid
        tree._has_root = None
        return tree

    # -- form conversions -----------------------------------------------------
    def _levels(self) -> list:
        """Sparse form (pending stores merged in); resolves the root flag."""
        if self._lv is None:
            pyr = self._host()
            self._lv = [None] + [_level_codes(pyr, l) for l in range(1, self.depth + 1)]
        if self._pend:
            codes = np.unique(np.asarray(self._pend, dtype=np.int64))
            self._pend = []
            L = self.depth
            self._lv = [None] + [np.union1d(self._lv[l], codes >> (3 * (L - l))) for l in range(1, L + 1)]
        if self._has_root is None:
            self._has_root = bool(self._lv[1].size)
        return self._lv

    def _host(self) -> np.ndarray:
        """Dense host pyramid (u32 words)."""
        if self._pyr is None:
            if self._lv is None:
                from . import _device
                self._pyr = _device.u32_to_numpy(self._dev).copy()
            else:
                lv = self._levels()
                pyr = np.zeros(_lib.pyramid_words(self.depth), dtype=np.uint32)
                for l in range(1, self.depth + 1):
                    if lv[l].size:
                        off = _lib.level_offset(l)
                        w = _codes_to_words(lv[l], l)
                        pyr[off:off + len(w)] = w
                self._pyr = pyr
        if self._has_root is None:
            self._has_root = bool(self._pyr[0] & 0xFF)
        return self._pyr

    def _device(self):
        """CUDA pyramid (int32 words), uploading the host copy if needed."""
        if self._dev is None:
            from . import _device
            self._dev = _device.to_device_u32(self._host())
        return self._dev

    def _root_flag(self) -> bool:
        if self._has_root is None:
            if self._lv is None and self._pyr is None and self._dev is not None:
                # device tree: the root exists iff level 1 (word 0) is non-empty -- one word, not the pyramid
                self._has_root = bool(int(self._dev[0].item()) & 0xFF)
            else:
                self._levels()
        return bool(self._has_root)

    def _mutate(self) -> None:
        """Before a mutation: keep only the sparse form."""
        self._levels()
        self._pyr = self._dev = self._bytes = None
        self._version += 1

    # -- reference API --------------------------------------------------------
    @property
    def root(self):
        return _NodeView(self, 0, 0) if self._root_flag() else None

    @root.setter
    def root(self, node) -> None:
        """Replace the whole tree by the subtree under ``node`` (``None``
        empties it), as the reference's ``merged.root = root`` (model.py:136).
        ``node`` is a view from an Octree or any object with a ``children``
        list of 8 (None = absent); nodes below ``depth`` are dropped."""
        L = self.depth
        if node is None:
            levels = [None] + [_EMPTY] * L
        elif isinstance(node, _NodeView):
            src, k, p = node._tree, node._level, node._prefix
            slv = src._levels()
            levels = [None]
            for j in range(1, L + 1):
                if k + j > src.depth:
                    levels.append(_EMPTY)
                    continue
                c = slv[k + j]
                lo, hi = np.searchsorted(c, [p << (3 * j), (p + 1) << (3 * j)])
                levels.append(c[lo:hi] - (p << (3 * j)))
        else:
            found = [[] for _ in range(L + 1)]
            stack = [(node, 0, 0)]
            while stack:
                n, lvl, code = stack.pop()
                if lvl == L:
                    continue
                for k, ch in enumerate(n.children):
                    if ch is not None:
                        found[lvl + 1].append(code * 8 + k)
                        stack.append((ch, lvl + 1, code * 8 + k))
            levels = [None] + [np.unique(np.asarray(f, dtype=np.int64)) for f in found[1:]]
        self._lv, self._pend = levels, []
        self._pyr = self._dev = self._bytes = None
        self._has_root = node is not None
        self._version += 1

    @property
    def is_empty(self) -> bool:
        return not self._root_flag()

    @property
    def node_count(self) -> int:
        lv = self._levels()
        if not self._has_root:
            return 0
        return 1 + sum(int(c.size) for c in lv[1:])

    def store(self, color: Color) -> None:
        """Insert a colour's path (octree.py:144-156).  Idempotent."""
        _check_color(color)
        r, g, b = color
        self.store_code(int(_SPREAD[0][r] | _SPREAD[1][g] | _SPREAD[2][b]) >> (3 * (8 - self.depth)))

    def store_code(self, code: int) -> None:
        """Insert a path given as a packed code (octree.py:158-169).  Like the
        reference walk ``(code >> shift) & 7``, only the low 3*depth bits of
        ``code`` (two's complement for negative ints) select the path."""
        code = int(code) & ((1 << (3 * self.depth)) - 1)
        if self._pyr is not None or self._dev is not None or self._bytes is not None:
            self._mutate()
        else:
            self._version += 1
        self._has_root = True
        self._pend.append(code)

    def _store_codes(self, codes) -> None:
        """Bulk insert of leaf codes (host)."""
        codes = np.asarray(codes, dtype=np.int64)
        if codes.size == 0:
            return
        self._mutate()
        self._has_root = True
        codes = np.unique(codes & ((1 << (3 * self.depth)) - 1))
        L = self.depth
        self._lv = [None] + [np.union1d(self._lv[l], codes >> (3 * (L - l))) for l in range(1, L + 1)]

    def contains(self, color: Color) -> bool:
        """True iff the full-depth path of ``color`` exists (octree.py:171-181)."""
        _check_color(color)
        r, g, b = color
        return self.contains_code(int(_SPREAD[0][r] | _SPREAD[1][g] | _SPREAD[2][b]) >> (3 * (8 - self.depth)))

    def contains_code(self, code: int) -> bool:
        """(octree.py:183-191); the low 3*depth bits of ``code`` select the path."""
        code = int(code) & ((1 << (3 * self.depth)) - 1)
        if self._lv is None and self._pyr is not None:
            pyr = self._host()
            if not self._has_root:
                return False
            return bool((int(pyr[_lib.level_offset(self.depth) + (code >> 5)]) >> (code & 31)) & 1)
        leaves = self._levels()[self.depth]
        if not self._has_root:
            return False
        i = int(np.searchsorted(leaves, code))
        return i < leaves.size and int(leaves[i]) == code

    def prune(self, new_depth: int) -> "Octree":
        """Copy truncated to ``new_depth`` levels (octree.py:193-204): the
        levels 1..new_depth; device-resident trees are pruned on the GPU
        (obg_prune)."""
        if not 1 <= new_depth <= self.depth:
            raise ValueError(f"new_depth must be in 1..{self.depth}, got {new_depth}")
        if self._lv is None and self._pyr is None and self._dev is not None:
            from . import _device
            out = _device.empty((_lib.pyramid_words(new_depth),), "int32")
            lib = _lib.load()
            _lib.check(lib.obg_prune(_device.ptr(self._dev), 1, self.depth, new_depth, _device.ptr(out),
                                     _device.stream_handle()))
            return Octree._from_device(out, new_depth)
        lv = self._levels()
        return Octree._from_levels([None] + [c.copy() for c in lv[1:new_depth + 1]], new_depth, self._has_root)

    def leaf_codes(self) -> list[int]:
        """Packed codes of all full-depth leaves, ascending (octree.py:206-211)."""
        return self.leaf_code_array().tolist()

    def leaf_code_array(self) -> np.ndarray:
        lv = self._levels()
        if not self._has_root:
            return np.zeros(0, dtype=np.int64)
        return lv[self.depth].copy()

    def leaf_colors(self) -> set[Color]:
        return {code_to_color(code, self.depth) for code in self.leaf_codes()}

    def to_bytes(self) -> bytes:
        """Preorder child-mask serialisation (octree.py:217-227, 258-267).

        Preorder is lexicographic order of node paths with a prefix before its
        extensions, i.e. ascending ``code << 3(L-l)`` with ties (a node and
        its all-zero-digit descendants) broken by level.  Device-resident
        trees are serialised on the GPU (obg_serialize)."""
        if self._bytes is not None and not self._pend:
            return self._bytes
        if self._lv is None and self._pyr is None and self._dev is not None:
            self._bytes = _serialize_device(self._dev, self.depth)
            if self._has_root is None:
                self._has_root = bool(self._bytes)
            return self._bytes
        lv = self._levels()
        if not self._has_root:
            return b""
        L = self.depth
        root = _child_masks(np.zeros(1, dtype=np.int64), lv[1]) if L >= 1 else np.zeros(1, np.uint8)
        keys = [np.zeros(1, dtype=np.int64)]
        vals = [root]
        for l in range(1, L + 1):
            c = lv[l]
            if c.size == 0:
                continue
            keys.append(((c << (3 * (L - l))) << 4) | l)
            vals.append(_child_masks(c, lv[l + 1]) if l < L else np.zeros(c.size, dtype=np.uint8))
        if len(keys) == 1:
            self._bytes = root.tobytes()
        else:
            order = np.argsort(np.concatenate(keys), kind="stable")
            self._bytes = np.concatenate(vals)[order].tobytes()
        return self._bytes

    @classmethod
    def from_bytes(cls, data: bytes, depth: int) -> "Octree":
        """Parse a :meth:`to_bytes` serialisation (octree.py:229-237)."""
        if not data:
            return cls(depth)
        tree, pos = decode_tree(data, 0, depth)
        if pos != len(data):
            raise FormatError("trailing data after octree", pos)
        tree._bytes = bytes(data)
        return tree

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, Octree):
            return NotImplemented
        if self.depth != other.depth:
            return False
        a, b = self._levels(), other._levels()
        # to_bytes is injective on (root flag, level sets) for a fixed depth
        return self._has_root == other._has_root and all(np.array_equal(x, y) for x, y in zip(a[1:], b[1:]))

    __hash__ = None  # mutable

    def __repr__(self) -> str:
        return f"<Octree depth={self.depth} nodes={self.node_count}>"


def _serialize_device(dev_pyramid, depth: int) -> bytes:
    """obg_serialize on the tree's CUDA pyramid; returns the host bytes."""
    import ctypes

    from . import _device
    lib = _lib.load()
    ws_bytes = lib.obg_serialize_workspace_bytes(depth)
    ws = _device.empty(((ws_bytes + 3) // 4,), "int32")
    cap = 1 + _lib.pyramid_words(depth) * 32
    out = _device.empty(((cap + 3) // 4,), "int32")
    n = ctypes.c_int64(0)
    _lib.check(lib.obg_serialize(_device.ptr(dev_pyramid), depth, 0, _device.ptr(out), cap, ctypes.byref(n),
                                 _device.ptr(ws), ws_bytes, _device.stream_handle()))
    if n.value == 0:
        return b""
    return _device.u32_to_numpy(out).view(np.uint8)[: n.value].tobytes()


def _decode_tree_native(data: bytes, pos: int, depth: int):
    import ctypes
    try:
        lib = _lib.load()
    except Exception:
        return None
    cap = max(len(data) - pos - 1, 0)
    codes = np.empty(max(cap, 1), dtype=np.uint32)
    levels = np.empty(max(cap, 1), dtype=np.uint8)
    n_nodes, end, off, kind = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int(0)
    buf = (ctypes.c_uint8 * len(data)).from_buffer_copy(data) if data else (ctypes.c_uint8 * 1)()
    rc = lib.obg_decode_tree_codes(buf, len(data), pos, depth, codes.ctypes.data, levels.ctypes.data, cap,
                                   ctypes.byref(n_nodes), ctypes.byref(end), ctypes.byref(off), ctypes.byref(kind))
    if rc == _lib.OBG_EFORMAT:
        if kind.value == 1:
            raise FormatError(f"octree node below leaf depth {depth}", off.value)
        raise FormatError("truncated octree data", off.value)
    if rc != _lib.OBG_OK:
        return None
    return _tree_from_preorder(codes[: n_nodes.value], levels[: n_nodes.value], depth), end.value


def _tree_from_preorder(codes: np.ndarray, levels: np.ndarray, depth: int) -> Octree:
    """Per-level code arrays from preorder (code, level) pairs: each level's
    codes are ascending in preorder, so a stable sort by level is the split."""
    order = np.argsort(levels, kind="stable")
    counts = np.bincount(levels, minlength=depth + 1)
    sorted_codes = codes[order].astype(np.int64)
    bounds = np.concatenate([[0], np.cumsum(counts[1:depth + 1])])
    lv = [None] + [sorted_codes[bounds[l - 1]:bounds[l]] for l in range(1, depth + 1)]
    return Octree._from_levels(lv, depth, has_root=True)


def decode_tree(data: bytes, pos: int, depth: int) -> tuple[Octree, int]:
    """Decode one non-empty tree starting at ``pos`` (octree.py:250-281).

    Iterative preorder walk with the reference's error order and offsets --
    native (obg_decode_tree_codes: O(nodes), a full depth-7 tree of 2.4 M
    nodes in ~10 ms instead of ~1 s) when libobg.so is loadable, else in
    Python."""
    _check_levels(depth)
    data = bytes(data) if not isinstance(data, (bytes, bytearray)) else data
    native = _decode_tree_native(data, pos, depth)
    tree, end = native if native is not None else _decode_tree_py(data, pos, depth)
    tree._bytes = bytes(data[pos:end])
    return tree, end


def _decode_tree_py(data: bytes, pos: int, depth: int) -> tuple[Octree, int]:
    n = len(data)
    codes, levels = [], []
    if pos >= n:
        raise FormatError("truncated octree data", pos)
    mask = data[pos]
    pos += 1
    stack = [(0, 0, mask)]
    while stack:
        level, prefix, rem = stack[-1]
        if rem == 0:
            stack.pop()
            continue
        low = rem & -rem
        stack[-1] = (level, prefix, rem ^ low)
        child_level, child = level + 1, prefix * 8 + low.bit_length() - 1
        if pos >= n:
            raise FormatError("truncated octree data", pos)
        m = data[pos]
        pos += 1
        if child_level == depth and m != 0:
            raise FormatError(f"octree node below leaf depth {depth}", pos - 1)
        codes.append(child)
        levels.append(child_level)
        stack.append((child_level, child, m))
    return _tree_from_preorder(np.asarray(codes, dtype=np.int64), np.asarray(levels, dtype=np.uint8), depth), pos
