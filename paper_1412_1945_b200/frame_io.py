"""Binary PPM frames / PGM masks and directory-backed frame sequences
(the frame-ingest side of the hot path).

Names, semantics, error messages and byte offsets follow the reference's
``frame_io.py`` (P6 frames with maxval 255, P5 masks of 0/255, sequences =
directories of ``.ppm`` files in name order).  Header parsing runs in the
native library (``obg_pnm_header``, host code -- no GPU needed), and whole
sequences are read by a pool of host threads straight into (pinned) memory
(``obg_read_pnm_files``) so the H2D copies of the classify pipeline can
start on them without another pass over the bytes; masks are written back by
``obg_write_pgm_masks`` the same way.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from pathlib import Path
from typing import Iterator

import numpy as np

from . import _lib
from .errors import FormatError


def _header(data: bytes, kind: int):
    lib = _lib.load()
    w, h, payload, off = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(-1)
    buf = ctypes.c_char_p(data)
    rc = lib.obg_pnm_header(ctypes.cast(buf, ctypes.c_void_p), len(data), kind, ctypes.byref(w), ctypes.byref(h),
                            ctypes.byref(payload), ctypes.byref(off))
    _lib.check(rc, off.value if off.value >= 0 else None)
    return int(w.value), int(h.value), int(payload.value)


def read_ppm(data: bytes) -> np.ndarray:
    """Decode a binary P6 PPM into an (h, w, 3) uint8 array."""
    data = bytes(data)
    w, h, payload = _header(data, 6)
    return np.frombuffer(data, dtype=np.uint8, count=w * h * 3, offset=payload).reshape(h, w, 3).copy()


def write_ppm(frame) -> bytes:
    frame = np.asarray(frame)
    if frame.ndim != 3 or frame.shape[2] != 3 or frame.dtype != np.uint8:
        raise ValueError(f"expected (h, w, 3) uint8 frame, got {frame.dtype} {frame.shape}")
    h, w = frame.shape[:2]
    return b"P6\n%d %d\n255\n" % (w, h) + np.ascontiguousarray(frame).tobytes()


def read_mask_pgm(data: bytes) -> np.ndarray:
    """Decode a binary P5 PGM of 0/255 values into an (h, w) bool mask."""
    data = bytes(data)
    w, h, payload = _header(data, 5)
    values = np.frombuffer(data, dtype=np.uint8, count=w * h, offset=payload)
    bad = (values != 0) & (values != 255)
    if bad.any():
        first = int(np.argmax(bad))
        raise FormatError(f"non-binary mask value {values[first]}", payload + first)
    return (values == 255).reshape(h, w)


def write_mask_pgm(mask) -> bytes:
    mask = np.asarray(mask)
    if mask.ndim != 2 or mask.dtype != bool:
        raise ValueError(f"expected (h, w) bool mask, got {mask.dtype} {mask.shape}")
    h, w = mask.shape
    return b"P5\n%d %d\n255\n" % (w, h) + np.where(mask, 255, 0).astype(np.uint8).tobytes()


def load_frame(path) -> np.ndarray:
    return read_ppm(Path(path).read_bytes())


def save_frame(path, frame) -> None:
    Path(path).write_bytes(write_ppm(frame))


def load_mask(path) -> np.ndarray:
    return read_mask_pgm(Path(path).read_bytes())


def save_mask(path, mask) -> None:
    Path(path).write_bytes(write_mask_pgm(mask))


def _paths_array(paths):
    enc = [str(p).encode() for p in paths]
    return (ctypes.c_char_p * len(enc))(*enc), enc


@dataclass
class FrameSequence:
    """An ordered directory of same-sized PPM frames."""

    directory: Path
    names: list
    width: int
    height: int

    @classmethod
    def scan(cls, directory) -> "FrameSequence":
        directory = Path(directory)
        names = sorted(p.name for p in directory.glob("*.ppm"))
        if not names:
            raise ValueError(f"no .ppm frames in {directory}")
        first = load_frame(directory / names[0])
        return cls(directory=directory, names=names, width=first.shape[1], height=first.shape[0])

    def __len__(self) -> int:
        return len(self.names)

    def path(self, index: int) -> Path:
        return self.directory / self.names[index]

    def items(self) -> Iterator:
        """Yield (file name, frame), checking each frame against the sequence size."""
        for name in self.names:
            frame = load_frame(self.directory / name)
            if frame.shape[:2] != (self.height, self.width):
                raise ValueError(f"frame {name} is {frame.shape[1]}x{frame.shape[0]}, "
                                 f"sequence is {self.width}x{self.height}")
            yield name, frame

    def frames(self) -> Iterator:
        for _, frame in self.items():
            yield frame

    def load_all(self) -> list:
        return list(self.frames())

    def load_batch(self, indices=None, out=None, pinned: bool = True, threads: int = 0):
        """Frames ``indices`` (default: all) as one (n, h, w, 3) uint8 array,
        read by ``threads`` host threads (0: all cores) straight into ``out``
        -- by default a new pinned torch tensor, the H2D source of the
        classify pipeline.  Same errors as ``items()``."""
        idx = list(range(len(self))) if indices is None else [int(i) for i in indices]
        shape = (len(idx), self.height, self.width, 3)
        if out is None:
            if pinned:
                from . import _device
                t = _device.torch()
                out = t.empty(shape, dtype=t.uint8, pin_memory=True)
            else:
                out = np.empty(shape, dtype=np.uint8)
        ptr = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
        if tuple(out.shape) != shape:
            raise ValueError(f"out must be {shape}")
        arr, _keep = _paths_array([self.path(i) for i in idx])
        bad, off = ctypes.c_int(-1), ctypes.c_int64(-1)
        rc = _lib.load().obg_read_pnm_files(arr, len(idx), 6, self.width, self.height, ptr, threads,
                                           ctypes.byref(bad), ctypes.byref(off))
        if rc != _lib.OBG_OK and rc == _lib.OBG_EINVAL and bad.value >= 0:
            # size mismatch: the reference's message names the file
            frame = load_frame(self.path(idx[bad.value]))
            raise ValueError(f"frame {self.names[idx[bad.value]]} is {frame.shape[1]}x{frame.shape[0]}, "
                             f"sequence is {self.width}x{self.height}")
        _lib.check(rc, off.value if off.value >= 0 else None)
        return out


def write_frame_sequence(directory, frames, start: int = 1) -> FrameSequence:
    """Write frames as ``frame_000001.ppm`` ... and return the scanned sequence."""
    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    for i, frame in enumerate(frames, start=start):
        save_frame(directory / f"frame_{i:06d}.ppm", frame)
    return FrameSequence.scan(directory)


def save_masks(masks, paths, threads: int = 0) -> None:
    """Write (n, h, w) masks (bool / uint8 nonzero = foreground; numpy or a
    CPU tensor) as 0/255 P5 PGM files, with ``threads`` host threads."""
    if hasattr(masks, "data_ptr"):
        if masks.is_cuda:
            raise ValueError("masks must be in host memory")
        m = masks.contiguous()
        n, h, w = (int(x) for x in m.shape)
        ptr = m.data_ptr()
    else:
        m = np.ascontiguousarray(masks)
        if m.dtype == bool:
            m = m.view(np.uint8)
        n, h, w = m.shape
        ptr = m.ctypes.data
    if len(paths) != n:
        raise ValueError(f"{len(paths)} paths for {n} masks")
    arr, _keep = _paths_array(paths)
    _lib.check(_lib.load().obg_write_pgm_masks(ptr, n, w, h, arr, threads))


def write_mask_sequence(directory, masks, names) -> list:
    """Write masks as PGMs named after the given frame basenames
    (reference ``frame_io.py:183-192``): ``<stem>.pgm`` per (mask, name) pair,
    pairs as ``zip`` forms them; returns the written file names.  Runs of
    same-shaped masks go to the threaded native writer (``save_masks``); the
    first mask that is not a 2-D bool array raises the reference's
    ``write_mask_pgm`` ValueError after the masks before it were written."""
    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    pairs = list(zip(masks, names))
    outs = [Path(name).stem + ".pgm" for _, name in pairs]
    arrays = []
    for m, _ in pairs:
        a = np.asarray(m)
        if a.ndim != 2 or a.dtype != bool:
            break
        arrays.append(a)
    start = 0
    while start < len(arrays):
        end = start + 1
        while end < len(arrays) and arrays[end].shape == arrays[start].shape:
            end += 1
        save_masks(np.stack(arrays[start:end]), [directory / o for o in outs[start:end]])
        start = end
    if len(arrays) < len(pairs):
        save_mask(directory / outs[len(arrays)], pairs[len(arrays)][0])   # raises
    return outs
