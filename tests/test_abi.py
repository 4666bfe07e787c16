"""The C-ABI library loads without a GPU and exports every symbol the public
header declares, with the documented size arithmetic and argument checks
(no device compute is issued here)."""

import ctypes
import os
import re

import pytest

from paper_1412_1945_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "obg.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(obg_\w+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.obg_abi_version() == _lib.ABI_VERSION


def test_size_helpers():
    lib = _lib.load()
    assert [lib.obg_pyramid_words(L) for L in range(1, 9)] == [1, 3, 19, 147, 1171, 9363, 74899, 599187]
    for L in range(1, 9):
        assert lib.obg_pyramid_words(L) == _lib.pyramid_words(L)
        assert lib.obg_cube_words(L) == _lib.cube_words(L)
        for l in range(1, L + 1):
            assert lib.obg_level_offset(L, l) == _lib.level_offset(l)
    assert lib.obg_pyramid_words(0) == -1 and lib.obg_pyramid_words(9) == -1
    assert lib.obg_build_workspace_bytes(64, 1, 6) == 64 * (8192 + 1184) * 4   # leaf cube + upper levels (padded)


@pytest.mark.parametrize("call", [
    lambda lib: lib.obg_build_presence(None, 4, 8, 8, 9, 1, 1, 1, None, None, None, 0, 0, None),
    lambda lib: lib.obg_build_presence(None, 0, 8, 8, 4, 1, 1, 1, None, None, None, 0, 0, None),
    lambda lib: lib.obg_build_presence(None, 2, 8, 8, 4, 1, 1, 3, None, None, None, 0, 0, None),
    lambda lib: lib.obg_classify(None, 1, 8, 8, 4, 0, 1, None, None, 0, None),
    lambda lib: lib.obg_classify(None, 1, 8, 8, 4, 1, 1, None, None, 7, None),
    lambda lib: lib.obg_merge(None, 0, 1, 4, 1, None, None, None),
    lambda lib: lib.obg_merge(None, 2, 1, 4, 0, None, None, None),
    lambda lib: lib.obg_prune(None, 1, 3, 4, None, None),
    lambda lib: lib.obg_pack_codes(None, 5, 0, None, None),
])
def test_invalid_arguments_rejected_before_device_work(call):
    lib = _lib.load()
    assert call(lib) == _lib.OBG_EINVAL
    assert lib.obg_last_error()
    with pytest.raises(ValueError):
        _lib.check(_lib.OBG_EINVAL)


def test_error_message_text():
    lib = _lib.load()
    lib.obg_build_presence(None, 2, 8, 8, 4, 1, 1, 3, None, None, None, 0, 0, None)
    assert b"need at least 3 frames for one group, got 2" in lib.obg_last_error()


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(_lib.LibraryNotBuilt):
        _lib.load()


@pytest.mark.parametrize("streaming", [0, 1])
def test_host_pool_copies(streaming):
    """obg_host_copy / obg_host_gather (the host copy pool, ordinary and
    non-temporal stores): any size, any destination alignment."""
    import numpy as np
    lib = _lib.load()
    rng = np.random.default_rng(7 + streaming)
    for size in (1, 15, 16, 17, 255, 4096, 262144, 262145, 1_000_003, 6_220_800):
        for off in (0, 1, 7, 16, 33):
            src = rng.integers(0, 256, size, dtype=np.uint8)
            dst = np.full(size + 64, 0xA5, np.uint8)
            assert lib.obg_host_copy(src.ctypes.data, size, dst.ctypes.data + off, streaming) == 0
            assert np.array_equal(dst[off:off + size], src)
            assert (dst[:off] == 0xA5).all() and (dst[off + size:] == 0xA5).all()   # nothing written outside
    blocks = [rng.integers(0, 256, 300_001, dtype=np.uint8) for _ in range(5)]
    dst = np.zeros(5 * 300_001 + 3, np.uint8)
    srcs = (ctypes.c_void_p * 5)(*[b.ctypes.data for b in blocks])
    assert lib.obg_host_gather(srcs, 5, 300_001, dst.ctypes.data + 3) == 0
    assert np.array_equal(dst[3:], np.concatenate(blocks))
    assert lib.obg_host_copy(None, 4, dst.ctypes.data, 0) != 0          # null source is an argument error
    assert lib.obg_host_copy(blocks[0].ctypes.data, 0, dst.ctypes.data, 1) == 0
