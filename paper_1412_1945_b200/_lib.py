"""ctypes binding of libobg.so, the sm_100a CUDA library behind every bulk op.

The library is built in-tree (``python -c "import __graft_entry__ as g;
g.build()"`` or ``make -C paper_1412_1945_b200/csrc``).  There is no CPU
fallback: if the library is missing every bulk entry point raises
:class:`LibraryNotBuilt`.  Host-only helpers (Octree scalar ops, model-file
parsing) do not need it.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# OBG_LIB_PATH: an alternative build of the same library (A/B kernel experiments, tools/ab.py)
LIB_PATH = os.environ.get("OBG_LIB_PATH") or os.path.join(_HERE, "_build", "libobg.so")

OBG_OK = 0
OBG_EINVAL = -1
OBG_EUNSUPPORTED = -2
OBG_ECUDA = -3
OBG_EFORMAT = -4
OBG_EIO = -5
WS_ZEROED = 1
MASK_U8 = 0
MASK_PACKED = 1
MASK_AFTER_MODEL = 0x100    # OBG_MASK_AFTER_MODEL: classify launched as a dependent of the model build

# Every symbol declared in include/obg.h, with its ctypes signature.
_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_int64
SIGNATURES = {
    "obg_abi_version": (_I, []),
    "obg_last_error": (ctypes.c_char_p, []),
    "obg_pyramid_words": (_L, [_I]),
    "obg_level_offset": (_L, [_I, _I]),
    "obg_cube_words": (_L, [_I]),
    "obg_build_workspace_bytes": (_L, [_I, _I, _I]),
    "obg_pack_codes": (_I, [_P, _L, _I, _P, _P]),
    "obg_build_presence": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _L, _I, _P]),
    "obg_build_model": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _L, _P, _P, _P, _P, _L, _I, _P]),
    "obg_pyramid_from_leaves": (_I, [_P, _I, _I, _P, _P]),
    "obg_prune": (_I, [_P, _I, _I, _I, _P, _P]),
    "obg_merge_counts": (_I, [_P, _I, _I, _I, _P, _P]),
    "obg_merge_threshold": (_I, [_P, _I, _I, _L, _P, _P, _P]),
    "obg_merge": (_I, [_P, _I, _I, _I, _L, _P, _P, _P]),
    "obg_leaf_cube": (_I, [_P, _I, _I, _P, _P]),
    "obg_classify": (_I, [_P, _I, _I, _I, _I, _I, _I, _P, _P, _I, _P]),
    "obg_classify_confusion": (_I, [_P, _I, _I, _I, _I, _I, _I, _P, _P, _I, _P, _P]),
    "obg_serialize_workspace_bytes": (_L, [_I]),
    "obg_serialize": (_I, [_P, _I, _I, _P, _L, ctypes.POINTER(ctypes.c_int64), _P, _L, _P]),
    "obg_pnm_header": (_I, [_P, _L, _I, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                            ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "obg_read_pnm_files": (_I, [ctypes.POINTER(ctypes.c_char_p), _I, _I, _L, _L, _P, _I,
                                ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64)]),
    "obg_write_pgm_masks": (_I, [_P, _I, _L, _L, ctypes.POINTER(ctypes.c_char_p), _I]),
    "obg_decode_tree": (_I, [_P, _L, _L, _I, _P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                             ctypes.POINTER(ctypes.c_int)]),
    "obg_decode_tree_codes": (_I, [_P, _L, _L, _I, _P, _P, _L, ctypes.POINTER(ctypes.c_int64),
                                   ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                   ctypes.POINTER(ctypes.c_int)]),
    "obg_host_gather": (_I, [ctypes.POINTER(ctypes.c_void_p), _I, _L, _P]),
    "obg_detect_host": (_I, [_P, _I, _I, _I, _I, _I, _I, _P, _P, _P]),
    "obg_host_copy": (_I, [_P, _L, _P, _I]),
    "obg_host_stage_release": (None, []),
    "obg_build_counts": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _L, _I, _P]),
    "obg_threshold_counts": (_I, [_P, _I, _I, _L, _P, _P, _P]),
    "obg_frame_diff": (_I, [_P, _P, _I, _L, _I, _P, _P]),
    "obg_running_average": (_I, [_P, _I, _L, _L, _P, _I, _P, _P]),
}
ABI_VERSION = 8


class LibraryNotBuilt(RuntimeError):
    pass


class ObgError(RuntimeError):
    pass


_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load libobg.so (once).  Raises LibraryNotBuilt if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LibraryNotBuilt(
                f"{LIB_PATH} is missing: build it with `python -c \"import __graft_entry__ as g; g.build()\"` "
                "(there is no CPU fallback for the octree hot path)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.obg_abi_version() != ABI_VERSION:
            raise LibraryNotBuilt(f"{LIB_PATH} ABI {lib.obg_abi_version()} != expected {ABI_VERSION}; rebuild it")
        _lib = lib
        return lib


def check(rc: int, offset: int | None = None) -> None:
    """Map a libobg status code to the reference's exception conventions
    (OBG_EFORMAT -> FormatError carrying the byte ``offset``)."""
    if rc == OBG_OK:
        return
    msg = load().obg_last_error().decode(errors="replace")
    if rc == OBG_EINVAL:
        raise ValueError(msg)
    if rc == OBG_EFORMAT:
        from .errors import FormatError
        raise FormatError(msg, offset)
    if rc == OBG_EIO:
        raise OSError(msg)
    raise ObgError(f"libobg error {rc}: {msg}")


def pyramid_words(levels: int) -> int:
    """Words in a per-level presence pyramid (pure arithmetic, no library)."""
    return sum(level_words(l) for l in range(1, levels + 1))


def level_words(level: int) -> int:
    return 1 if level <= 1 else 1 << (3 * level - 5)


def level_offset(level: int) -> int:
    return sum(level_words(m) for m in range(1, level))


def cube_words(levels: int) -> int:
    """Words of one region's classify operand: the leaf cube, plus for L = 7
    a 2-bit state per L=6 cell (16384 words), 32 words of cell counts
    (k_l7_states; the L7 classify picks its path by them) and one bit per
    L=6 cell whose 8 leaves are all present (8192 words)."""
    return level_words(levels) + (16384 + 32 + 8192 if levels == 7 else 0)
