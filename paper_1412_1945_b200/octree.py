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
# pyramid helpers (host side)
# ---------------------------------------------------------------------------
def _level_bits(pyr: np.ndarray, level: int) -> np.ndarray:
    """Level ``level`` of a pyramid as a bool array of 8**level entries."""
    off, nw = _lib.level_offset(level), _lib.level_words(level)
    bits = np.unpackbits(pyr[off:off + nw].view(np.uint8), bitorder="little")
    return bits[: 8 ** level].astype(bool)


def _level_bytes(pyr: np.ndarray, level: int) -> np.ndarray:
    off, nw = _lib.level_offset(level), _lib.level_words(level)
    return pyr[off:off + nw].view(np.uint8)


class _NodeView:
    """Read-only stand-in for the reference's ``_Node`` (octree.py:106-110)."""

    __slots__ = ("_tree", "_level", "_prefix")

    def __init__(self, tree: "Octree", level: int, prefix: int):
        self._tree, self._level, self._prefix = tree, level, prefix

    @property
    def children(self) -> list:
        t = self._tree
        if self._level >= t.depth:
            return [None] * 8
        pyr = t._host()
        mask = int(_level_bytes(pyr, self._level + 1)[self._prefix])
        return [_NodeView(t, self._level + 1, self._prefix * 8 + k) if mask >> k & 1 else None
                for k in range(8)]


class Octree:
    """Presence tree over quantized colours, leaves at a fixed depth (octree.py:113-247)."""

    __slots__ = ("depth", "_pyr", "_dev", "_has_root", "_version")

    def __init__(self, depth: int):
        _check_levels(depth)
        self.depth = depth
        self._pyr: np.ndarray | None = np.zeros(_lib.pyramid_words(depth), dtype=np.uint32)
        self._dev = None              # optional CUDA copy of the pyramid (int32 words)
        self._has_root: bool | None = False   # None: derive from level 1 (device trees)
        self._version = 0

    # -- construction from pyramids ------------------------------------------
    @classmethod
    def _from_pyramid(cls, pyramid: np.ndarray, depth: int, has_root: bool | None = None) -> "Octree":
        tree = cls(depth)
        tree._pyr = np.ascontiguousarray(pyramid, dtype=np.uint32).copy()
        if len(tree._pyr) != _lib.pyramid_words(depth):
            raise ValueError("pyramid size does not match depth")
        tree._has_root = bool(tree._pyr[0] & 0xFF) if has_root is None else bool(has_root)
        return tree

    @classmethod
    def _from_device(cls, dev_pyramid, depth: int) -> "Octree":
        """Tree backed by a CUDA pyramid (GPU build/merge output).  Its root
        exists iff level 1 is non-empty, which holds for built trees
        (model.py:93-109) and merged trees (model.py:133-136)."""
        tree = cls(depth)
        tree._pyr = None
        tree._dev = dev_pyramid
        tree._has_root = None
        return tree

    def _host(self) -> np.ndarray:
        if self._pyr is None:
            from . import _device
            self._pyr = _device.u32_to_numpy(self._dev).copy()
        if self._has_root is None:
            self._has_root = bool(self._pyr[0] & 0xFF)
        return self._pyr

    def _device(self):
        """CUDA pyramid (int32 words), uploading the host copy if needed."""
        if self._dev is None:
            from . import _device
            self._dev = _device.to_device_u32(self._host())
        return self._dev

    def _mutate(self) -> np.ndarray:
        pyr = self._host()
        self._dev = None
        self._version += 1
        return pyr

    # -- reference API --------------------------------------------------------
    @property
    def root(self):
        self._host()
        return _NodeView(self, 0, 0) if self._has_root else None

    @property
    def is_empty(self) -> bool:
        self._host()
        return not self._has_root

    @property
    def node_count(self) -> int:
        pyr = self._host()
        if not self._has_root:
            return 0
        return 1 + int(np.unpackbits(pyr.view(np.uint8)).sum())

    def store(self, color: Color) -> None:
        """Insert a colour's path (octree.py:144-156).  Idempotent."""
        _check_color(color)
        r, g, b = color
        self.store_code(int(_SPREAD[0][r] | _SPREAD[1][g] | _SPREAD[2][b]) >> (3 * (8 - self.depth)))

    def store_code(self, code: int) -> None:
        """Insert a path given as a packed code (octree.py:158-169)."""
        pyr = self._mutate()
        self._has_root = True
        for level in range(1, self.depth + 1):
            p = code >> (3 * (self.depth - level))
            pyr[_lib.level_offset(level) + (p >> 5)] |= np.uint32(1 << (p & 31))

    def _store_codes(self, codes) -> None:
        """Bulk insert (host; used for small trees built from Python data)."""
        codes = np.unique(np.asarray(codes, dtype=np.int64))
        if codes.size == 0:
            return
        pyr = self._mutate()
        self._has_root = True
        for level in range(1, self.depth + 1):
            p = codes >> (3 * (self.depth - level))
            words = np.zeros(_lib.level_words(level), dtype=np.uint32)
            np.bitwise_or.at(words, p >> 5, (np.uint32(1) << (p & 31).astype(np.uint32)))
            off = _lib.level_offset(level)
            pyr[off:off + len(words)] |= words

    def contains(self, color: Color) -> bool:
        """True iff the full-depth path of ``color`` exists (octree.py:171-181)."""
        _check_color(color)
        r, g, b = color
        return self.contains_code(int(_SPREAD[0][r] | _SPREAD[1][g] | _SPREAD[2][b]) >> (3 * (8 - self.depth)))

    def contains_code(self, code: int) -> bool:
        """(octree.py:183-191)"""
        pyr = self._host()
        if not self._has_root:
            return False
        off = _lib.level_offset(self.depth)
        return bool((int(pyr[off + (code >> 5)]) >> (code & 31)) & 1)

    def prune(self, new_depth: int) -> "Octree":
        """Copy truncated to ``new_depth`` levels (octree.py:193-204).

        On the pyramid this keeps levels 1..new_depth; device-resident trees
        are pruned on the GPU (obg_prune)."""
        if not 1 <= new_depth <= self.depth:
            raise ValueError(f"new_depth must be in 1..{self.depth}, got {new_depth}")
        if self._pyr is None and self._dev is not None:
            from . import _device
            out = _device.empty((_lib.pyramid_words(new_depth),), "int32")
            lib = _lib.load()
            _lib.check(lib.obg_prune(_device.ptr(self._dev), 1, self.depth, new_depth, _device.ptr(out),
                                     _device.stream_handle()))
            return Octree._from_device(out, new_depth)
        pyr = self._host()
        return Octree._from_pyramid(pyr[: _lib.pyramid_words(new_depth)], new_depth, self._has_root)

    def leaf_codes(self) -> list[int]:
        """Packed codes of all full-depth leaves, ascending (octree.py:206-211)."""
        return self.leaf_code_array().tolist()

    def leaf_code_array(self) -> np.ndarray:
        pyr = self._host()
        if not self._has_root:
            return np.zeros(0, dtype=np.int64)
        return np.flatnonzero(_level_bits(pyr, self.depth)).astype(np.int64)

    def leaf_colors(self) -> set[Color]:
        return {code_to_color(code, self.depth) for code in self.leaf_codes()}

    def to_bytes(self) -> bytes:
        """Preorder child-mask serialisation (octree.py:217-227).

        Node (l, p) lands at preorder position
            1 + sum_{1<=m<l} (rank_m(p >> 3(l-m)) + 1) + sum_{m>=l} rank_m(p << 3(m-l))
        where rank_m(q) counts level-m nodes with code < q; its byte is byte p
        of level l+1 (0 for leaves)."""
        pyr = self._host()
        if not self._has_root:
            return b""
        L = self.depth
        bits = [None] + [_level_bits(pyr, l) for l in range(1, L + 1)]
        excl = [None] + [np.cumsum(b, dtype=np.int64) - b for b in bits[1:]]
        total = 1 + sum(int(b.sum()) for b in bits[1:])
        out = np.zeros(total, dtype=np.uint8)
        out[0] = _level_bytes(pyr, 1)[0]
        for l in range(1, L + 1):
            p = np.flatnonzero(bits[l]).astype(np.int64)
            if p.size == 0:
                continue
            pos = np.ones_like(p)
            for m in range(1, l):
                pos += excl[m][p >> (3 * (l - m))] + 1
            for m in range(l, L + 1):
                pos += excl[m][p << (3 * (m - l))]
            if l < L:
                out[pos] = _level_bytes(pyr, l + 1)[p]
        return out.tobytes()

    @classmethod
    def from_bytes(cls, data: bytes, depth: int) -> "Octree":
        """Parse a :meth:`to_bytes` serialisation (octree.py:229-237)."""
        if not data:
            return cls(depth)
        tree, pos = decode_tree(data, 0, depth)
        if pos != len(data):
            raise FormatError("trailing data after octree", pos)
        return tree

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, Octree):
            return NotImplemented
        if self.depth != other.depth:
            return False
        a, b = self._host(), other._host()
        # to_bytes is injective on (root flag, pyramid) for a fixed depth
        return self._has_root == other._has_root and np.array_equal(a, b)

    __hash__ = None  # mutable

    def __repr__(self) -> str:
        return f"<Octree depth={self.depth} nodes={self.node_count}>"


def _decode_tree_native(data: bytes, pos: int, depth: int):
    import ctypes
    try:
        lib = _lib.load()
    except Exception:
        return None
    pyr = np.zeros(_lib.pyramid_words(depth), dtype=np.uint32)
    end, off, kind = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int(0)
    buf = (ctypes.c_uint8 * len(data)).from_buffer_copy(data) if data else (ctypes.c_uint8 * 1)()
    rc = lib.obg_decode_tree(buf, len(data), pos, depth, pyr.ctypes.data, ctypes.byref(end), ctypes.byref(off),
                             ctypes.byref(kind))
    if rc == _lib.OBG_EFORMAT:
        if kind.value == 1:
            raise FormatError(f"octree node below leaf depth {depth}", off.value)
        raise FormatError("truncated octree data", off.value)
    if rc != _lib.OBG_OK:
        return None
    return Octree._from_pyramid(pyr, depth, has_root=True), end.value


def decode_tree(data: bytes, pos: int, depth: int) -> tuple[Octree, int]:
    """Decode one non-empty tree starting at ``pos`` (octree.py:250-281).

    Iterative preorder walk with the reference's error order and offsets --
    native (obg_decode_tree, ~100x faster: a full depth-7 tree of 2.4 M nodes
    in ~10 ms instead of ~1 s) when libobg.so is loadable, else in Python."""
    _check_levels(depth)
    data = bytes(data) if not isinstance(data, (bytes, bytearray)) else data
    native = _decode_tree_native(data, pos, depth)
    if native is not None:
        return native
    return _decode_tree_py(data, pos, depth)


def _decode_tree_py(data: bytes, pos: int, depth: int) -> tuple[Octree, int]:
    n = len(data)
    codes = [[] for _ in range(depth + 1)]
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
        codes[child_level].append(child)
        stack.append((child_level, child, m))
    pyr = np.zeros(_lib.pyramid_words(depth), dtype=np.uint32)
    for level in range(1, depth + 1):
        if not codes[level]:
            continue
        p = np.asarray(codes[level], dtype=np.int64)
        words = np.zeros(_lib.level_words(level), dtype=np.uint32)
        np.bitwise_or.at(words, p >> 5, np.uint32(1) << (p & 31).astype(np.uint32))
        off = _lib.level_offset(level)
        pyr[off:off + len(words)] = words
    return Octree._from_pyramid(pyr, depth, has_root=True), pos
