"""Host-side logic of the drop-in package (no GPU): Octree pyramid semantics,
serialisation, validation messages, k_min, model files.  Expected values are
the reference's own KATs (reference tests/test_octree.py, test_model.py) and
the oracle."""

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import paper_1412_1945_b200 as obg
from paper_1412_1945_b200 import FormatError, ModelConfig, Octree
from oracle import octree_oracle as orc

channels = st.integers(0, 255)
colors = st.tuples(channels, channels, channels)
levels_st = st.integers(1, 8)


def tree_of(cols, levels):
    t = Octree(levels)
    for c in cols:
        t.store(c)
    return t


def test_child_index_kat(golden):
    assert [obg.child_index((200, 100, 50), b) for b in range(7, -1, -1)] == \
        golden["kat"]["child_index_200_100_50"]
    assert obg.child_index((255, 0, 0), 7) == 4


def test_quantize_and_code_roundtrip():
    assert obg.quantize_color((200, 100, 50), 4) == (192, 96, 48)
    assert obg.quantize_color((255, 255, 255), 2) == (192, 192, 192)
    with pytest.raises(ValueError):
        obg.quantize_color((0, 0, 0), 9)
    for L in range(1, 9):
        c = (17, 93, 241)
        assert obg.code_to_color(obg.pack_code(c, L), L) == obg.quantize_color(c, L)


def test_store_kats(golden):
    t = tree_of([(255, 255, 255)], 1)
    assert t.leaf_codes() == [7] and t.node_count == 2
    t = tree_of([(0, 0, 0), (0, 0, 0)], 4)
    assert t.node_count == 5
    t = tree_of([(0, 0, 0), (255, 255, 255)], 2)
    kat = golden["kat"]["store_bw_d2"]
    assert t.node_count == kat["nodes"] and t.leaf_codes() == kat["leaves"]
    assert t.to_bytes().hex() == kat["bytes"]
    assert tree_of([(255, 255, 255)], 2).to_bytes() == bytes([0x80, 0x80, 0x00])
    assert Octree(4).to_bytes() == b"" and Octree.from_bytes(b"", 4).is_empty


def test_prune_kats(golden):
    t = tree_of([(192, 96, 48)], 4)
    p = t.prune(2)
    assert p.depth == 2
    assert sorted(p.leaf_colors()) == [tuple(c) for c in golden["kat"]["prune_4_to_2_leaf_colors"]]
    assert p.contains((200, 100, 50))
    assert Octree(4).prune(2).is_empty
    with pytest.raises(ValueError):
        Octree(3).prune(4)
    with pytest.raises(ValueError):
        Octree(3).prune(0)


def test_root_only_tree():
    t = Octree.from_bytes(b"\x00", 3)
    assert not t.is_empty and t.node_count == 1 and t.leaf_codes() == []
    assert t.to_bytes() == b"\x00"
    assert t.prune(1).to_bytes() == b"\x00"
    assert t != Octree(3)


def test_from_bytes_errors():
    t = tree_of([(8, 8, 8)], 3)
    data = t.to_bytes()
    with pytest.raises(FormatError) as e:
        Octree.from_bytes(data[:-1], 3)
    assert e.value.offset == len(data) - 1
    with pytest.raises(FormatError) as e:
        Octree.from_bytes(data + b"\x00", 3)
    assert e.value.offset == len(data)
    with pytest.raises(FormatError) as e:
        Octree.from_bytes(tree_of([(0, 0, 0)], 2).to_bytes(), 1)
    assert e.value.offset == 1


def _random_oracle_tree(rng, depth, dead_ends):
    n = int(rng.integers(0, 60))
    codes = rng.integers(0, 8 ** depth, size=n)
    if not dead_ends:
        return orc.tree_from_codes(codes, depth)
    trees = [orc.tree_from_codes(rng.integers(0, 8 ** depth, size=int(rng.integers(0, 40))), depth)
             for _ in range(int(rng.integers(1, 6)))]
    return orc.merge_trees(trees, float(rng.choice([0.2, 0.4, 0.5, 0.7])), depth)


def _octree_from_oracle(t):
    return Octree.from_bytes(orc.to_bytes(t), t.depth)


@pytest.mark.parametrize("seed", range(40))
def test_to_bytes_matches_oracle(seed):
    rng = np.random.default_rng(seed)
    depth = int(rng.integers(1, 9))
    t = _random_oracle_tree(rng, depth, dead_ends=seed % 2 == 1)
    want = orc.to_bytes(t)
    ours = _octree_from_oracle(t)
    assert ours.to_bytes() == want
    assert ours.node_count == t.node_count()
    assert ours.leaf_codes() == t.leaf_codes()
    for nd in range(1, depth + 1):
        assert ours.prune(nd).to_bytes() == orc.to_bytes(orc.prune(t, nd))


@settings(max_examples=60, deadline=None)
@given(st.lists(colors, max_size=30), levels_st)
def test_store_roundtrip_property(stored, levels):
    t = tree_of(stored, levels)
    assert Octree.from_bytes(t.to_bytes(), levels) == t
    codes = [obg.pack_code(c, levels) for c in stored]
    assert t.to_bytes() == orc.to_bytes(orc.tree_from_codes(codes, levels))
    for c in stored:
        assert t.contains(c)
    assert 1 + levels <= t.node_count <= 1 + levels * max(1, len(set(codes))) or not stored


@settings(max_examples=40, deadline=None)
@given(st.lists(colors, min_size=1, max_size=30), st.integers(2, 8), st.data())
def test_prune_quantize_commutation(stored, depth, data):
    new_depth = data.draw(st.integers(1, depth))
    probe = data.draw(colors)
    t = tree_of(stored, depth)
    q = lambda c, L: obg.quantize_color(c, L)  # noqa: E731
    assert t.prune(new_depth).contains(probe) == any(q(s, new_depth) == q(probe, new_depth) for s in stored)


def test_node_view_children():
    t = tree_of([(0, 0, 0), (255, 255, 255)], 2)
    kids = t.root.children
    assert [k is not None for k in kids] == [True] + [False] * 6 + [True]
    assert kids[7].children[7] is not None and kids[7].children[7].children == [None] * 8


def test_k_min_matches_reference_decisions(golden):
    for key, want in golden["kat"]["k_min"].items():
        n, th = key.split(":")
        assert obg.merge_k_min(int(n), float(th)) == want, key
    # exhaustive against the reference's float test
    for n in range(1, 400):
        for th in (0.1, 0.3, 0.55, 0.57, 0.58, 0.6, 0.7, 0.9, 1.0, 1.0 / n, 0.5):
            want = min(k for k in range(1, n + 1) if k / n >= th)
            assert obg.merge_k_min(n, th) == want


@pytest.mark.parametrize("kwargs", [
    {"levels": 0}, {"levels": 9}, {"threshold": 0.0}, {"threshold": 1.5},
    {"grid_rows": 0}, {"group_size": 0}, {"group_size": 5, "training_frames": 4},
])
def test_invalid_configs_rejected(kwargs):
    with pytest.raises(ValueError):
        ModelConfig(**kwargs)


def test_region_helpers():
    assert obg.region_of(0, 0, 64, 48, 3, 5) == (0, 0)
    assert obg.region_of(99, 99, 100, 100, 2, 2) == (1, 1)
    assert obg.region_of(45, 30, 90, 60, 3, 3) == (1, 1)
    for extent in range(1, 40):
        for parts in range(1, 7):
            b = obg.region_bounds(extent, parts)
            assert b == orc.region_bounds(extent, parts)
            for v in range(extent):
                p = min(parts - 1, v * parts // extent)
                assert b[p] <= v < b[p + 1]


def test_validation_messages_without_gpu():
    # argument errors surface before any device work (reference model.py:78-101)
    with pytest.raises(ValueError, match="no frames given"):
        obg.build_background_model([], ModelConfig())
    with pytest.raises(ValueError, match="need at least 3 frames"):
        obg.build_background_model([np.zeros((2, 2, 3), np.uint8)] * 2, ModelConfig(group_size=3, training_frames=3))
    with pytest.raises(ValueError, match="does not match first frame"):
        obg.build_background_model([np.zeros((2, 2, 3), np.uint8), np.zeros((2, 3, 3), np.uint8)], ModelConfig())
    with pytest.raises(ValueError, match="expected a group of 1 frames"):
        obg.build_frame_tree([np.zeros((2, 2, 3), np.uint8)] * 2, (0, 0), ModelConfig())
    with pytest.raises(ValueError, match="outside 1x1 grid"):
        obg.build_frame_tree([np.zeros((2, 2, 3), np.uint8)], (1, 0), ModelConfig())
    with pytest.raises(ValueError, match="no trees to merge"):
        obg.merge_trees([], 0.5, 2)
    with pytest.raises(ValueError, match="does not match levels"):
        obg.merge_trees([Octree(2), Octree(3)], 0.5, 2)
    with pytest.raises(ValueError, match="threshold must be in"):
        obg.merge_trees([Octree(2)], 0.0, 2)
    m = obg.BackgroundModel(ModelConfig(), 4, 4, trees=[[Octree(4)]])
    with pytest.raises(ValueError, match="model expects 4x4"):
        obg.detect_octree(m, np.zeros((4, 5, 3), np.uint8))
    with pytest.raises(ValueError, match="uint8 frame"):
        obg.detect_octree(m, np.zeros((4, 4, 3), np.int16))
    with pytest.raises(ValueError, match="uint8 pixels"):
        obg.pack_codes(np.zeros((4, 2), np.uint8), 4)


def test_model_file_roundtrip_host(golden):
    rng = np.random.default_rng(43)
    trees = [[tree_of([tuple(int(v) for v in rng.integers(0, 256, 3)) for _ in range(20)], 4) for _ in range(3)]
             for _ in range(2)]
    trees[1][2] = Octree(4)
    model = obg.BackgroundModel(ModelConfig(levels=4, threshold=0.3, grid_rows=2, grid_cols=3, training_frames=8),
                                frame_width=14, frame_height=10, trees=trees)
    blob = obg.write_model(model)
    restored = obg.read_model(blob)
    assert obg.write_model(restored) == blob
    assert restored.trees[1][2].is_empty
    for r in range(2):
        for c in range(3):
            assert restored.trees[r][c] == model.trees[r][c]
    bad = bytearray(blob)
    bad[:4] = b"NOPE"
    with pytest.raises(FormatError):
        obg.read_model(bytes(bad))
    bad = bytearray(blob)
    bad[4] = 99
    with pytest.raises(FormatError):
        obg.read_model(bytes(bad))
    with pytest.raises(FormatError):
        obg.read_model(blob[:-1])
    with pytest.raises(FormatError):
        obg.read_model(blob + b"\x00")


@pytest.mark.parametrize("case", range(0, 96, 5))
def test_golden_model_files_parse(golden, case):
    """Reference-written OBGM files parse and re-serialise byte-identically."""
    blob = bytes.fromhex(golden["random_cases"][case]["model_file"])
    assert obg.write_model(obg.read_model(blob)) == blob


def test_native_decode_tree_matches_python_walk():
    """obg_decode_tree (native) vs the Python preorder walk on valid trees,
    truncations and corrupted bytes: same pyramid and end position, or the
    same FormatError message and offset."""
    from paper_1412_1945_b200 import _lib
    from paper_1412_1945_b200.errors import FormatError
    from paper_1412_1945_b200.octree import _decode_tree_native, _decode_tree_py
    try:
        _lib.load()
    except Exception:
        pytest.skip("libobg.so not built")
    rng = np.random.default_rng(99)
    for case in range(300):
        depth = int(rng.integers(1, 6))
        codes = rng.integers(0, 8 ** depth, size=int(rng.integers(1, 40)))
        from oracle import octree_oracle as orc
        blob = bytearray(orc.to_bytes(orc.tree_from_codes(codes, depth)))
        kind = case % 4
        if kind == 1:
            blob = blob[: int(rng.integers(0, len(blob)))]
        elif kind == 2 and len(blob) > 1:
            blob[int(rng.integers(0, len(blob)))] = int(rng.integers(0, 256))
        elif kind == 3:
            blob += bytes(rng.integers(0, 256, size=3).astype(np.uint8))
        data = bytes(blob)
        results = []
        for fn in (_decode_tree_native, _decode_tree_py):
            try:
                tree, end = fn(data, 0, depth)
                results.append(("ok", tree._host().tobytes(), end))
            except FormatError as e:
                results.append(("err", str(e), e.offset))
        assert results[0] == results[1], (case, results)


def test_store_code_masks_digits_like_reference():
    """Reference store_code/contains_code walk ``(code >> shift) & 7``
    (octree.py:158-191): only the low 3*depth bits select the path, for
    negative and oversized codes alike; a call never half-mutates the tree."""
    t = Octree(3)
    t.store_code(-1)
    assert t.leaf_codes() == [511] and t.to_bytes().hex() == "80808000"
    t = Octree(3)
    t.store_code(8 ** 3 + 5)
    assert t.leaf_codes() == [5] and t.contains_code(5) and t.contains_code(8 ** 3 + 5)
    assert t.node_count == 4 and not t.contains_code(6)


def test_root_assignment():
    """``tree.root = other.root`` / ``= None`` (the reference assigns
    ``merged.root = root``, model.py:136)."""
    a = Octree(3)
    for c in ((0, 0, 0), (255, 0, 128), (9, 200, 77)):
        a.store(c)
    b = Octree(3)
    b.root = a.root
    assert b == a and b.to_bytes() == a.to_bytes()
    b.root = None
    assert b.is_empty and b.to_bytes() == b"" and b.node_count == 0
    # a subtree view: the level-1 child of a's first colour, re-rooted
    sub = next(ch for ch in a.root.children if ch is not None)
    c = Octree(2)
    c.root = sub
    assert c.leaf_codes() == sorted({code & 63 for code in a.leaf_codes() if code >> 6 == sub._prefix})
    # any object with a ``children`` list of 8 (e.g. the reference's _Node)
    class N:
        def __init__(self, kids=None):
            self.children = kids or [None] * 8
    leaf = N()
    d = Octree(2)
    d.root = N([None, N([leaf] + [None] * 7)] + [None] * 6)
    assert d.leaf_codes() == [8] and d.node_count == 3


def test_sparse_tree_ops_are_cheap():
    """O(nodes) host trees: a 2-colour depth-8 round trip well under the
    reference property test's 200 ms deadline (tests/test_octree.py:238-247)."""
    import time
    t0 = time.perf_counter()
    for _ in range(20):
        t = Octree(8)
        t.store((255, 255, 255))
        t.store((1, 2, 3))
        data = t.to_bytes()
        r = Octree.from_bytes(data, 8)
        assert r == t and r.to_bytes() == data and r.node_count == 17
    assert (time.perf_counter() - t0) / 20 < 0.02


def test_frames_validation_without_gpu():
    from paper_1412_1945_b200 import _device
    for bad in (np.zeros((2, 4, 4), np.uint8), np.zeros((2, 4, 4, 4), np.uint8), np.zeros((2, 4, 4, 3), np.int16)):
        with pytest.raises(ValueError):
            _device.frames_on_device(bad)
