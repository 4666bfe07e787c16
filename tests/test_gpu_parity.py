"""GPU parity: the CUDA path (through libobg.so's C ABI) against the reference's
recorded outputs (tests/golden/golden.json) and the CPU oracle.  Integer /
byte / index work throughout, so every comparison is bit-exact."""

import numpy as np
import pytest

import paper_1412_1945_b200 as obg
from cases import random_case_inputs
from helpers import mask_digest, mask_hex, sha
from oracle import octree_oracle as orc
from paper_1412_1945_b200 import ModelConfig, Octree, _lib

pytestmark = pytest.mark.gpu


def _cfg(rec, n):
    return ModelConfig(levels=rec["levels"], threshold=rec["threshold"], grid_rows=rec["grid_rows"],
                       grid_cols=rec["grid_cols"], group_size=rec["group_size"], training_frames=n)


def test_library_loaded_from_tree(cuda):
    lib = _lib.load()
    assert lib._name.endswith("paper_1412_1945_b200/_build/libobg.so")


@pytest.mark.parametrize("levels", range(1, 9))
def test_pack_codes(cuda, levels):
    rng = np.random.default_rng(levels)
    px = rng.integers(0, 256, size=(37, 29, 3), dtype=np.uint8)
    assert np.array_equal(obg.pack_codes(px, levels), orc.pack_codes(px, levels))


def test_pack_codes_kat(cuda, golden):
    rng = np.random.default_rng(7)
    px = rng.integers(0, 256, size=(13, 9, 3), dtype=np.uint8)
    for L, want in golden["kat"]["pack_codes_13x9"].items():
        assert obg.pack_codes(px, int(L)).ravel().tolist() == want


@pytest.mark.parametrize("case", range(96))
def test_random_case(cuda, golden, case):
    rec = golden["random_cases"][case]
    x = random_case_inputs(case)
    frames = list(x["frames"])
    cfg = _cfg(rec, len(frames))
    R, C, gs = cfg.grid_rows, cfg.grid_cols, cfg.group_size
    for g in range(len(frames) // gs):
        for r in range(R):
            for c in range(C):
                t = obg.build_frame_tree(frames[g * gs:(g + 1) * gs], (r, c), cfg)
                assert t.to_bytes().hex() == rec["group_trees"][g][r][c]
    model = obg.build_background_model(frames, cfg)
    for r in range(R):
        for c in range(C):
            assert model.trees[r][c].to_bytes().hex() == rec["merged"][r][c]
    for nd, want in rec["pruned00"].items():
        assert model.trees[0][0].prune(int(nd)).to_bytes().hex() == want
    for probe, want in zip(x["probes"], rec["masks"]):
        assert mask_hex(obg.detect_octree(model, probe)) == want
    assert obg.write_model(model).hex() == rec["model_file"]
    # merge of host-side trees (the reference's merge_trees API)
    groups = [obg.build_frame_tree(frames[g * gs:(g + 1) * gs], (0, 0), cfg) for g in range(len(frames) // gs)]
    host = [Octree.from_bytes(t.to_bytes(), cfg.levels) for t in groups]
    assert obg.merge_trees(host, cfg.threshold, cfg.levels).to_bytes().hex() == rec["merged"][0][0]


@pytest.mark.parametrize("case", range(96))
def test_loaded_model_detect(cuda, golden, case):
    """The reference's ``octabg detect`` flow (cli.py:181-187): a model FILE
    written by the reference -> read_model -> detect_octree per frame (and
    batched), against the reference's masks.  The trees come from bytes on
    the host, so the host tree -> obg_leaf_cube -> classify path is pinned."""
    rec = golden["random_cases"][case]
    x = random_case_inputs(case)
    model = obg.read_model(bytes.fromhex(rec["model_file"]))
    for r in range(rec["grid_rows"]):
        for c in range(rec["grid_cols"]):
            assert model.trees[r][c].to_bytes().hex() == rec["merged"][r][c]
    for probe, want in zip(x["probes"], rec["masks"]):
        assert mask_hex(obg.detect_octree(model, probe)) == want
    batch = obg.detect_octree_batch(model, x["probes"])
    for i, want in enumerate(rec["masks"]):
        assert mask_hex(batch[i]) == want
    assert obg.write_model(model).hex() == rec["model_file"]


@pytest.mark.parametrize("case", range(0, 96, 7))
def test_counts(cuda, golden, case):
    rec = golden["random_cases"][case]
    x = random_case_inputs(case)
    dev = cuda.from_numpy(np.ascontiguousarray(x["frames"][:1])).cuda()
    _, cnt = obg.build_presence(dev, rec["levels"], counts=True)
    assert sha(cnt[0, 0].cpu().numpy().astype(np.int64)) == rec["counts0_sha"]


def _check_config(rec, scene, cuda, packed_too=False):
    assert sha(scene.train) == rec["train_sha"] and sha(scene.test) == rec["test_sha"]
    cfg = ModelConfig(levels=rec["levels"], threshold=rec["threshold"], training_frames=len(scene.train))
    train = cuda.from_numpy(scene.train).cuda()
    model = obg.build_background_model_device(train, cfg)
    blob = model.trees[0][0].to_bytes()
    assert len(blob) == rec["merged_len"] and sha(blob) == rec["merged_sha"]
    assert model.trees[0][0].node_count == rec["merged_nodes"]
    pyr, cnt = obg.build_presence(train[: len(rec["frame_trees"])], cfg.levels, counts=True)
    for i, ft in enumerate(rec["frame_trees"]):
        t = Octree._from_device(pyr[i, 0], cfg.levels)
        assert sha(t.to_bytes()) == ft["sha"]
        assert sha(np.asarray(t.leaf_codes(), dtype=np.int64)) == ft["leaf_sha"]
    assert sha(cnt[0, 0].cpu().numpy().astype(np.int64)) == rec["counts0_sha"]
    chunk = 32
    for s in range(0, len(scene.test), chunk):
        frames = cuda.from_numpy(scene.test[s:s + chunk]).cuda()
        masks = obg.classify(model, frames).cpu().numpy()
        for i in range(len(masks)):
            assert int(masks[i].sum()) == rec["mask_fg"][s + i], f"frame {s + i}"
            assert mask_digest(masks[i]) == rec["mask_sha"][s + i], f"frame {s + i}"
        if packed_too:
            packed = obg.classify(model, frames, packed=True).cpu().numpy()
            want = np.packbits(masks.reshape(len(masks), -1).astype(bool), axis=1, bitorder="little")
            assert np.array_equal(packed, want)
        del frames


@pytest.mark.parametrize("cid", [0, 1, 2, 3])
def test_config(cuda, golden, cid):
    from paper_1412_1945_b200 import scenes
    rec = next(r for r in golden["configs"] if r["config"] == cid)
    _check_config(rec, scenes.generate(cid), cuda, packed_too=cid in (0, 3))


@pytest.mark.parametrize("variant", ["constant", "uniform"])
@pytest.mark.parametrize("levels", [4, 5, 6, 7])
def test_config4(cuda, golden, variant, levels):
    from paper_1412_1945_b200 import scenes
    rec = next(r for r in golden["configs"] if r["config"] == 4 and r["variant"] == variant
               and r["levels"] == levels and not r.get("extra"))
    _check_config(rec, scenes.generate(4, levels=levels, variant=variant), cuda)


def test_config4_partial_l7(cuda, golden):
    """C4 uniform 4K at L7 with threshold 1.0 (tests/golden/make_golden.py
    EXTRA_JOBS): a merged tree with about half of the 2^21 leaves, so the
    masks are about half foreground and the L7 state table holds mostly
    partially filled cells -- the thr-0.5 record is a full cube."""
    from paper_1412_1945_b200 import scenes
    rec = next(r for r in golden["configs"] if r.get("extra") and r["levels"] == 7 and r["variant"] == "uniform")
    assert 0.2 < rec["merged_leaves"] / 8 ** 7 < 0.8
    assert 0.2 < sum(rec["mask_fg"]) / (len(rec["mask_fg"]) * rec["width"] * rec["height"]) < 0.8
    _check_config(rec, scenes.generate(4, levels=7, variant="uniform"), cuda)


# --- reference behaviours (reference tests/test_detect.py, test_model.py) ------------
def uniform(h, w, color):
    return np.full((h, w, 3), color, dtype=np.uint8)


def test_training_frame_is_all_background(cuda):
    rng = np.random.default_rng(5)
    frame = rng.integers(0, 256, size=(12, 16, 3), dtype=np.uint8)
    model = obg.build_background_model([frame] * 20, ModelConfig(training_frames=20))
    assert not obg.detect_octree(model, frame).any()


def test_single_deviating_pixel(cuda):
    frame = uniform(10, 10, (128, 128, 128))
    model = obg.build_background_model([frame] * 10, ModelConfig(training_frames=10))
    probe = frame.copy()
    probe[3, 7] = (0, 0, 0)
    mask = obg.detect_octree(model, probe)
    assert mask[3, 7] and mask.sum() == 1 and mask.dtype == np.bool_


def test_empty_region_tree_flags_everything(cuda):
    frames = [uniform(6, 6, (0, 0, 0)), uniform(6, 6, (255, 255, 255))]
    model = obg.build_background_model(frames, ModelConfig(threshold=1.0, training_frames=2))
    assert model.trees[0][0].is_empty
    assert obg.detect_octree(model, uniform(6, 6, (0, 0, 0))).all()


def test_static_foreground_absorption(cuda):
    background = np.full((20, 20, 3), (30, 30, 30), dtype=np.uint8)
    with_object = background.copy()
    with_object[5:10, 5:10] = (200, 60, 60)
    frames = [with_object] * 30 + [background] * 70
    absorbed = obg.build_background_model(frames, ModelConfig(levels=4, threshold=0.25))
    rejected = obg.build_background_model(frames, ModelConfig(levels=4, threshold=0.5))
    assert absorbed.trees[0][0].contains((200, 60, 60))
    assert not rejected.trees[0][0].contains((200, 60, 60))
    assert absorbed.trees[0][0].contains((30, 30, 30)) and rejected.trees[0][0].contains((30, 30, 30))


def test_trailing_partial_group_discarded(cuda):
    rng = np.random.default_rng(37)
    frames = [rng.integers(0, 256, size=(4, 4, 3), dtype=np.uint8) for _ in range(7)]
    cfg = ModelConfig(levels=3, threshold=0.5, group_size=3, training_frames=7)
    model = obg.build_background_model(frames, cfg)
    trees = [obg.build_frame_tree(g, (0, 0), cfg) for g in (frames[0:3], frames[3:6])]
    assert model.trees[0][0] == obg.merge_trees(trees, 0.5, 3)


def test_training_frames_cap(cuda):
    rng = np.random.default_rng(3)
    frames = [rng.integers(0, 256, size=(8, 8, 3), dtype=np.uint8) for _ in range(9)]
    a = obg.build_background_model(frames, ModelConfig(levels=3, threshold=0.4, training_frames=5))
    b = obg.build_background_model(frames[:5], ModelConfig(levels=3, threshold=0.4, training_frames=5))
    assert a.trees[0][0] == b.trees[0][0]


# --- edge cases of the kernels' fast / generic paths -----------------------------------
@pytest.mark.parametrize("shape", [(1, 1), (1, 16), (3, 7), (16, 1), (5, 48), (17, 33), (64, 64)])
@pytest.mark.parametrize("levels", [1, 2, 6, 7, 8])
def test_shapes_and_levels(cuda, shape, levels):
    rng = np.random.default_rng(hash((shape, levels)) % 2 ** 32)
    h, w = shape
    base = rng.integers(0, 256, size=(1, 1, 1, 3))
    frames = np.clip(base + rng.integers(-20, 21, size=(9, h, w, 3)), 0, 255).astype(np.uint8)
    probes = np.clip(base + rng.integers(-30, 31, size=(5, h, w, 3)), 0, 255).astype(np.uint8)
    cfg = ModelConfig(levels=levels, threshold=0.4, training_frames=9)
    model = obg.build_background_model(list(frames), cfg)
    want = orc.build_background_model(list(frames), levels, 0.4)
    assert model.trees[0][0].to_bytes() == orc.to_bytes(want[(0, 0)])
    masks = obg.detect_octree_batch(model, probes)
    for i in range(len(probes)):
        assert np.array_equal(masks[i], orc.detect_octree(want, probes[i], levels))
    packed = obg.classify(model, cuda.from_numpy(probes).cuda(), packed=True).cpu().numpy()
    want_packed = np.packbits(masks.reshape(len(masks), -1), axis=1, bitorder="little")
    assert np.array_equal(packed, want_packed)


def test_misaligned_views_take_generic_path(cuda):
    rng = np.random.default_rng(11)
    big = rng.integers(0, 256, size=(6 * 32 * 32 * 3 + 5,), dtype=np.uint8)
    dev = cuda.from_numpy(big).cuda()
    frames = dev[5:].view(6, 32, 32, 3)          # 5-byte offset: not 16-byte aligned
    host = big[5:].reshape(6, 32, 32, 3)
    cfg = ModelConfig(levels=5, threshold=0.5, training_frames=6)
    model = obg.build_background_model_device(frames, cfg)
    want = orc.build_background_model(list(host), 5, 0.5)
    assert model.trees[0][0].to_bytes() == orc.to_bytes(want[(0, 0)])
    masks = obg.classify(model, frames).cpu().numpy()
    for i in range(6):
        assert np.array_equal(masks[i].astype(bool), orc.detect_octree(want, host[i], 5))


@pytest.mark.parametrize("grid", [(1, 1), (2, 2), (3, 1), (1, 5), (7, 9)])
@pytest.mark.parametrize("gs", [1, 2, 3])
def test_grids_and_groups(cuda, grid, gs):
    rng = np.random.default_rng(grid[0] * 100 + grid[1] * 10 + gs)
    frames = rng.integers(0, 256, size=(8, 6, 10, 3), dtype=np.uint8) // 64 * 64
    cfg = ModelConfig(levels=3, threshold=0.5, grid_rows=grid[0], grid_cols=grid[1], group_size=gs,
                      training_frames=8)
    model = obg.build_background_model(list(frames), cfg)
    want = orc.build_background_model(list(frames), 3, 0.5, grid[0], grid[1], gs)
    for r in range(grid[0]):
        for c in range(grid[1]):
            assert model.trees[r][c].to_bytes() == orc.to_bytes(want[(r, c)]), (r, c)
    probe = rng.integers(0, 256, size=(6, 10, 3), dtype=np.uint8) // 64 * 64
    assert np.array_equal(obg.detect_octree(model, probe), orc.detect_octree(want, probe, 3, grid[0], grid[1]))


def test_device_serializer_matches_host(cuda):
    import ctypes
    from paper_1412_1945_b200 import _device
    lib = _lib.load()
    rng = np.random.default_rng(99)
    for levels in range(1, 9):
        for trial in range(3):
            trees = [orc.tree_from_codes(rng.integers(0, 8 ** levels, size=int(rng.integers(0, 300))), levels)
                     for _ in range(5)]
            merged = orc.merge_trees(trees, 0.4, levels) if trial else trees[0]
            want = orc.to_bytes(merged)
            t = Octree.from_bytes(want, levels) if want else Octree(levels)
            dev = t._device()
            ws_bytes = lib.obg_serialize_workspace_bytes(levels)
            ws = _device.empty((ws_bytes // 4,), "int32")
            out = _device.empty((t.node_count + 1,), "uint8")
            n = ctypes.c_int64(0)
            _lib.check(lib.obg_serialize(_device.ptr(dev), levels, int(not t.is_empty), _device.ptr(out),
                                         out.numel(), ctypes.byref(n), _device.ptr(ws), ws_bytes,
                                         _device.stream_handle()))
            assert out[: n.value].cpu().numpy().tobytes() == want


def test_pyramid_from_leaves_and_prune(cuda):
    from paper_1412_1945_b200 import _device
    lib = _lib.load()
    rng = np.random.default_rng(5)
    for levels in range(1, 9):
        codes = rng.integers(0, 8 ** levels, size=500)
        t = orc.tree_from_codes(codes, levels)
        leaves = np.zeros(_lib.level_words(levels), dtype=np.uint32)
        np.bitwise_or.at(leaves, codes >> 5, np.uint32(1) << (codes & 31).astype(np.uint32))
        dev_leaves = _device.to_device_u32(leaves)
        out = _device.empty((_lib.pyramid_words(levels),), "int32")
        _lib.check(lib.obg_pyramid_from_leaves(_device.ptr(dev_leaves), 1, levels, _device.ptr(out),
                                               _device.stream_handle()))
        tree = Octree._from_device(out, levels)
        assert tree.to_bytes() == orc.to_bytes(t)
        for nd in range(1, levels + 1):
            assert tree.prune(nd).to_bytes() == orc.to_bytes(orc.prune(t, nd))


def test_merge_counts_and_threshold(cuda):
    from paper_1412_1945_b200 import _device
    lib = _lib.load()
    rng = np.random.default_rng(8)
    levels, n = 4, 11
    trees = [obg.build_frame_tree([rng.integers(0, 256, size=(9, 9, 3), dtype=np.uint8)], (0, 0),
                                  ModelConfig(levels=levels)) for _ in range(n)]
    pyr = cuda.stack([t._device() for t in trees]).unsqueeze(1).contiguous()
    pw = _lib.pyramid_words(levels)
    counts = _device.empty((1, pw * 32), "int32")
    _lib.check(lib.obg_merge_counts(_device.ptr(pyr), n, 1, levels, _device.ptr(counts), _device.stream_handle()))
    want_counts = sum(np.unpackbits(t._host().view(np.uint8), bitorder="little").astype(np.int64) for t in trees)
    assert np.array_equal(counts.cpu().numpy()[0], want_counts)
    for k_min in (1, 3, 6, 11):
        out = _device.empty((1, pw), "int32")
        cube = _device.empty((1, _lib.cube_words(levels)), "int32")
        _lib.check(lib.obg_merge_threshold(_device.ptr(counts), 1, levels, k_min, _device.ptr(out),
                                           _device.ptr(cube), _device.stream_handle()))
        fused, fused_cube = obg.merge_pyramids(pyr, levels, k_min, with_cube=True)
        assert cuda.equal(out, fused) and cuda.equal(cube, fused_cube)
        ref_cube = _device.empty((1, _lib.cube_words(levels)), "int32")
        _lib.check(lib.obg_leaf_cube(_device.ptr(out), 1, levels, _device.ptr(ref_cube), _device.stream_handle()))
        assert cuda.equal(cube, ref_cube)


@pytest.mark.parametrize("levels", range(1, 9))
def test_fused_merge_cube_matches_leaf_cube(cuda, levels):
    from paper_1412_1945_b200 import _device
    lib = _lib.load()
    rng = np.random.default_rng(levels + 40)
    trees = [orc.tree_from_codes(rng.integers(0, 8 ** levels, size=int(rng.integers(1, 3000))), levels)
             for _ in range(7)]
    pyr = cuda.stack([Octree.from_bytes(orc.to_bytes(t), levels)._device() for t in trees]).unsqueeze(1)
    for k_min in (1, 2, 4, 7):
        merged, cube = obg.merge_pyramids(pyr.contiguous(), levels, k_min, with_cube=True)
        ref_cube = _device.empty((1, _lib.cube_words(levels)), "int32")
        _lib.check(lib.obg_leaf_cube(_device.ptr(merged), 1, levels, _device.ptr(ref_cube), _device.stream_handle()))
        assert cuda.equal(cube, ref_cube)
        want = orc.merge_trees(trees, k_min / 7 - 1e-12, levels)
        assert Octree._from_device(merged[0], levels).to_bytes() == orc.to_bytes(want)


@pytest.mark.parametrize("n_trees", [1, 7, 8, 9, 255, 2015, 2017, 2100])
def test_merge_many_trees(cuda, n_trees):
    """SWAR byte counters and their 32-bit spill path (> 2016 trees)."""
    rng = np.random.default_rng(n_trees)
    levels = 2
    trees = [orc.tree_from_codes(rng.integers(0, 64, size=int(rng.integers(0, 12))), levels) for _ in range(n_trees)]
    pyr = cuda.stack([(Octree.from_bytes(orc.to_bytes(t), levels) if t.root else Octree(levels))._device()
                      for t in trees]).unsqueeze(1).contiguous()
    for thr in (1.0 / n_trees, 0.1, 0.19, 0.5, 1.0):
        merged = obg.merge_pyramids(pyr, levels, obg.merge_k_min(n_trees, thr))
        want = orc.merge_trees(trees, thr, levels)
        assert Octree._from_device(merged[0], levels).to_bytes() == orc.to_bytes(want), thr


def test_captured_step_matches_eager(cuda, golden):
    """CUDA-graph replay of build + classify (the bench's steady state)."""
    from paper_1412_1945_b200 import scenes
    from paper_1412_1945_b200.pipeline import CapturedStep
    rec = next(r for r in golden["configs"] if r["config"] == 1)
    sc = scenes.generate(1, n_test=24)
    train, test = cuda.from_numpy(sc.train).cuda(), cuda.from_numpy(sc.test).cuda()
    cfg = ModelConfig(levels=rec["levels"], threshold=rec["threshold"], training_frames=len(sc.train))
    step = CapturedStep(train, test, cfg)
    for _ in range(3):
        masks = step.step().cpu().numpy()
        assert sha(step.model.trees[0][0].to_bytes()) == rec["merged_sha"]
        for i in range(len(masks)):
            assert mask_digest(masks[i]) == rec["mask_sha"][i]
    # different training frames: the model views of the next replays must see
    # the new trees (no stale host caches), for both graphs
    old_model = step.model
    old_bytes = old_model.trees[0][0].to_bytes()
    half = len(sc.train) // 2
    alt = np.concatenate([sc.train[half:], sc.test[: len(sc.train) - half]])
    train.copy_(cuda.from_numpy(alt).cuda())
    want_alt = orc.to_bytes(orc.build_background_model(list(alt), rec["levels"], rec["threshold"])[(0, 0)])
    assert want_alt != old_bytes
    for replay in (step.step, step.build):
        replay()
        assert step.model.trees[0][0].to_bytes() == want_alt
        assert obg.write_model(step.model) == obg.write_model(obg.build_background_model(list(alt), cfg))
    train.copy_(cuda.from_numpy(sc.train).cuda())
    step.step()
    # new frames copied into the static input: the replays classify them --
    # the one-graph step and the split build / classify graphs alike
    test.copy_(cuda.from_numpy(sc.train[:24]).cuda())
    eager = obg.classify(step.model, test).clone()
    assert cuda.equal(step.step(), eager)
    step.build()
    assert sha(step.model.trees[0][0].to_bytes()) == rec["merged_sha"]
    assert cuda.equal(step.classify(), eager)
    want = orc.build_background_model(list(sc.train), rec["levels"], rec["threshold"])
    for i in range(0, 24, 6):
        assert np.array_equal(eager[i].cpu().numpy().astype(bool), orc.detect_octree(want, sc.train[i], rec["levels"]))


def test_process_batches_pipeline(cuda, golden):
    """Overlapped host->device->host pipeline (the bench's e2e path)."""
    from paper_1412_1945_b200 import scenes
    from paper_1412_1945_b200.pipeline import process_batches
    rec = next(r for r in golden["configs"] if r["config"] == 1)
    sc = scenes.generate(1, n_test=37)
    cfg = ModelConfig(levels=rec["levels"], threshold=rec["threshold"], training_frames=len(sc.train))
    train = cuda.from_numpy(sc.train).pin_memory()
    test = cuda.from_numpy(sc.test).pin_memory()
    for chunk in (8, 16, 64):
        model, masks = process_batches(train, test, cfg, chunk=chunk)
        cuda.cuda.synchronize()
        assert sha(model.trees[0][0].to_bytes()) == rec["merged_sha"]
        m = masks.numpy()
        for i in range(37):
            assert mask_digest(m[i]) == rec["mask_sha"][i], (chunk, i)
    model, packed = process_batches(train, test, cfg, chunk=16, packed=True)
    cuda.cuda.synchronize()
    assert np.array_equal(packed.numpy(), np.packbits(m.reshape(37, -1).astype(bool), axis=1, bitorder="little"))


def test_build_model_abi_and_workspace_contract(cuda):
    """obg_build_model == build_presence + merge, and the build workspace is
    handed back all-zero (what lets callers skip clearing it)."""
    from paper_1412_1945_b200 import _device
    from paper_1412_1945_b200.model import _WORKSPACES
    lib = _lib.load()
    rng = np.random.default_rng(77)
    # every build flavour: flat shared-bitset K1 (L <= 6, levels at its flush),
    # global-bitset K1 + k_levels_cube (L >= 7, generic grids / odd sizes)
    for levels, (h, w), grid in [(6, (48, 64), (1, 1)), (5, (33, 20), (2, 3)), (7, (32, 32), (1, 1)),
                                 (3, (16, 16), (1, 1)), (8, (16, 16), (1, 1)), (1, (16, 16), (1, 1)),
                                 (2, (20, 12), (2, 2)), (4, (64, 32), (1, 1)), (6, (9, 13), (1, 1))]:
        base = rng.integers(0, 256, size=(1, 1, 1, 3))
        frames = np.clip(base + rng.integers(-30, 31, size=(10, h, w, 3)), 0, 255).astype(np.uint8)
        dev = cuda.from_numpy(frames).cuda()
        cfg = ModelConfig(levels=levels, threshold=0.4, grid_rows=grid[0], grid_cols=grid[1], training_frames=10)
        model = obg.build_background_model_device(dev, cfg)
        want = orc.build_background_model(list(frames), levels, 0.4, grid[0], grid[1])
        for r in range(grid[0]):
            for c in range(grid[1]):
                assert model.trees[r][c].to_bytes() == orc.to_bytes(want[(r, c)])
        pyr = obg.build_presence(dev, levels, grid[0], grid[1])
        merged, cube = obg.merge_pyramids(pyr, levels, obg.merge_k_min(10, 0.4), with_cube=True)
        assert cuda.equal(merged, model._dev_pyr) and cuda.equal(cube, model._dev_cube)
        cuda.cuda.synchronize()
        for ws in _WORKSPACES.values():
            assert int(ws.count_nonzero()) == 0
    # a caller-owned workspace (what a captured graph uses) is handed back zeroed too
    from paper_1412_1945_b200.model import new_workspace
    ws = new_workspace(lib.obg_build_workspace_bytes(10, 1, 6))
    frames = rng.integers(0, 256, size=(10, 48, 64, 3), dtype=np.uint8)
    cfg = ModelConfig(levels=6, threshold=0.4, training_frames=10)
    model = obg.build_background_model_device(cuda.from_numpy(frames).cuda(), cfg, workspace=ws)
    assert model.trees[0][0].to_bytes() == orc.to_bytes(orc.build_background_model(list(frames), 6, 0.4)[(0, 0)])
    cuda.cuda.synchronize()
    assert int(ws.count_nonzero()) == 0
    with pytest.raises(ValueError):
        obg.build_background_model_device(cuda.from_numpy(frames).cuda(), cfg, workspace=ws[:4])


@pytest.mark.gpu
def test_build_model_groups_and_repeat(cuda):
    """Groups of frames per tree (segments of a CTA end mid-range), a dropped
    trailing partial group, and back-to-back builds reusing the kept
    workspace (zero-on-return)."""
    rng = np.random.default_rng(5)
    for levels, gs in [(6, 3), (5, 2), (7, 4)]:
        frames = rng.integers(0, 256, size=(11, 40, 64, 3), dtype=np.uint8)
        frames[:, :20] = frames[0, :20]                      # half of each frame static
        dev = cuda.from_numpy(frames).cuda()
        cfg = ModelConfig(levels=levels, threshold=0.5, group_size=gs, training_frames=11)
        want = orc.build_background_model(list(frames), levels, 0.5, group_size=gs)
        for _ in range(3):
            model = obg.build_background_model_device(dev, cfg)
            assert model.trees[0][0].to_bytes() == orc.to_bytes(want[(0, 0)])


@pytest.mark.gpu
def test_build_model_many_trees(cuda):
    """> 16 x 252 trees per merge: the byte counters of k_merge_fused (16 tree
    groups) spill into the 32-bit shared counters (the `wide` path); levels 3-7
    cover its block-0 levels and tile levels."""
    rng = np.random.default_rng(8)
    n = 4100
    base = rng.integers(0, 256, size=(1, 1, 1, 3))
    frames = np.clip(base + rng.integers(-40, 41, size=(n, 8, 16, 3)), 0, 255).astype(np.uint8)
    for levels, thr in [(4, 0.5), (5, 0.05), (3, 0.99), (7, 0.02)]:
        cfg = ModelConfig(levels=levels, threshold=thr, training_frames=n)
        model = obg.build_background_model_device(cuda.from_numpy(frames).cuda(), cfg)
        want = orc.build_background_model(list(frames), levels, thr)
        assert model.trees[0][0].to_bytes() == orc.to_bytes(want[(0, 0)])


@pytest.mark.gpu
@pytest.mark.parametrize("grid", [(2, 3), (3, 5), (4, 1), (1, 6), (5, 7)])
@pytest.mark.parametrize("levels", [3, 5, 6])
def test_region_grid_band_classify(cuda, grid, levels):
    """Region grids with W % 16 == 0 take the band kernels (one bitset /
    operand per column region in shared memory, units cut by a column
    boundary per pixel): merged trees (groups of 1 and 2), a per-region frame
    tree, masks (u8 and bit-packed) and fused confusion counts against the
    oracle."""
    rng = np.random.default_rng(levels * 100 + grid[0] * 10 + grid[1])
    h, w = 50, 96
    base = rng.integers(0, 256, size=(1, h, w, 3))
    train = np.clip(base + rng.integers(-20, 21, size=(9, h, w, 3)), 0, 255).astype(np.uint8)
    probe = np.clip(base + rng.integers(-40, 41, size=(5, h, w, 3)), 0, 255).astype(np.uint8)
    probe[:, 5:30, 10:70] = rng.integers(0, 256, size=3).astype(np.uint8)
    R, C = grid
    cfg = ModelConfig(levels=levels, threshold=0.5, grid_rows=R, grid_cols=C, training_frames=9)
    model = obg.build_background_model(list(train), cfg)
    want_model = orc.build_background_model(list(train), levels, 0.5, R, C)
    for r in range(R):                       # band build kernel: every region's merged tree
        for c in range(C):
            assert model.trees[r][c].to_bytes() == orc.to_bytes(want_model[(r, c)]), (r, c)
    # groups of 2 frames + per-frame trees (obg_build_presence through the band kernel)
    cfg2 = ModelConfig(levels=levels, threshold=0.5, grid_rows=R, grid_cols=C, group_size=2, training_frames=9)
    m2 = obg.build_background_model(list(train), cfg2)
    w2 = orc.build_background_model(list(train), levels, 0.5, R, C, group_size=2)
    for r in range(R):
        for c in range(C):
            assert m2.trees[r][c].to_bytes() == orc.to_bytes(w2[(r, c)]), ("group 2", r, c)
    pyr = obg.build_presence(cuda.from_numpy(train[:3]).cuda(), levels, R, C, 1)
    for g in range(3):
        for r, c in ((0, 0), (R - 1, C // 2), (R // 2, C - 1)):
            want = orc.build_frame_tree([train[g]], (r, c), levels, R, C)
            assert Octree._from_device(pyr[g, r * C + c], levels).to_bytes() == orc.to_bytes(want), (g, r, c)
    dev = cuda.from_numpy(probe).cuda()
    masks = obg.classify(model, dev).cpu().numpy()
    packed = obg.classify(model, dev, packed=True).cpu().numpy()
    truth = (rng.random((5, h, w)) < 0.4).astype(np.uint8)
    counts = obg.classify_confusion(model, dev, cuda.from_numpy(truth).cuda())
    tn = tp = fn = fp = 0
    for i in range(len(probe)):
        want = orc.detect_octree(want_model, probe[i], levels, R, C)
        assert np.array_equal(masks[i].astype(bool), want), i
        assert np.array_equal(np.unpackbits(packed[i], bitorder="little")[: h * w].astype(bool), want.ravel()), i
        t = truth[i].astype(bool)
        tp += int((want & t).sum()); fp += int((want & ~t).sum())
        fn += int((~want & t).sum()); tn += int((~want & ~t).sum())
    assert (counts.true_neg, counts.true_pos, counts.false_neg, counts.false_pos) == (tn, tp, fn, fp)


@pytest.mark.gpu
@pytest.mark.parametrize("levels,grid,gs", [(4, (1, 1), 1), (5, (1, 1), 2), (6, (1, 1), 1), (6, (2, 3), 1), (3, (3, 2), 2)])
def test_sharded_build_counts(cuda, levels, grid, gs):
    """The multi-GPU build path on one GPU: obg_build_counts on two shards,
    the counts summed as the NCCL all-reduce would, obg_threshold_counts with
    the global k_min -> every region's merged tree equals the reference's merge
    of all frames; build_background_model_sharded (no process group) likewise."""
    from paper_1412_1945_b200 import _device
    from paper_1412_1945_b200.distributed import build_background_model_sharded
    rng = np.random.default_rng(levels * 31 + gs)
    h, w = 40, 64
    base = rng.integers(0, 256, size=(1, h, w, 3))
    frames = np.clip(base + rng.integers(-30, 31, size=(12, h, w, 3)), 0, 255).astype(np.uint8)
    R, C = grid
    thr = 0.5
    cfg = ModelConfig(levels=levels, threshold=thr, grid_rows=R, grid_cols=C, group_size=gs, training_frames=12)
    want = orc.build_background_model(list(frames), levels, thr, R, C, group_size=gs)
    lib = _lib.load()
    pw = _lib.pyramid_words(levels)
    total = cuda.zeros((R * C, pw * 32), dtype=cuda.int32, device="cuda")
    for shard in (frames[:6], frames[6:]):
        dev = cuda.from_numpy(np.ascontiguousarray(shard)).cuda()
        counts = cuda.empty((R * C, pw * 32), dtype=cuda.int32, device="cuda")
        ng = len(shard) // gs
        wsb = lib.obg_build_workspace_bytes(ng, R * C, levels)
        ws = cuda.zeros((wsb + 3) // 4, dtype=cuda.int32, device="cuda")
        _lib.check(lib.obg_build_counts(_device.ptr(dev), ng * gs, h, w, levels, R, C, gs, _device.ptr(counts),
                                        _device.ptr(ws), wsb, _lib.WS_ZEROED, _device.stream_handle()))
        assert int(ws.abs().sum()) == 0            # workspace handed back zeroed
        total += counts
    k_min = obg.merge_k_min(12 // gs, thr)
    merged = cuda.empty((R * C, pw), dtype=cuda.int32, device="cuda")
    cube = cuda.empty((R * C, _lib.cube_words(levels)), dtype=cuda.int32, device="cuda")
    _lib.check(lib.obg_threshold_counts(_device.ptr(total), R * C, levels, k_min, _device.ptr(merged),
                                        _device.ptr(cube), _device.stream_handle()))
    model = obg.BackgroundModel(cfg, frame_width=w, frame_height=h, _device_pyramids=merged, _device_cube=cube)
    single = build_background_model_sharded(cuda.from_numpy(frames).cuda(), cfg)
    for r in range(R):
        for c in range(C):
            assert model.trees[r][c].to_bytes() == orc.to_bytes(want[(r, c)]), (r, c)
            assert single.trees[r][c].to_bytes() == orc.to_bytes(want[(r, c)]), (r, c)
    probe = frames[3]
    assert np.array_equal(obg.detect_octree(model, probe), orc.detect_octree(want, probe, levels, R, C))


def test_device_entry_points_validate_inputs(cuda):
    """classify / classify_confusion / build_presence / the device build take
    raw pointers: strided views are made contiguous, host tensors are copied
    over, malformed shapes / dtypes raise ValueError before any launch."""
    rng = np.random.default_rng(31)
    frames = rng.integers(0, 256, size=(6, 24, 40, 3), dtype=np.uint8)
    cfg = ModelConfig(levels=5, threshold=0.5, training_frames=6)
    model = obg.build_background_model(list(frames), cfg)
    dev = cuda.from_numpy(frames).cuda()
    want = obg.classify(model, dev).cpu()
    wide = cuda.from_numpy(np.concatenate([frames, frames], axis=2)).cuda()
    strided = wide[:, :, :40]                      # non-contiguous view of the same pixels
    assert not strided.is_contiguous()
    assert cuda.equal(obg.classify(model, strided).cpu(), want)
    assert cuda.equal(obg.classify(model, cuda.from_numpy(frames)).cpu(), want)   # CPU tensor in
    assert cuda.equal(obg.build_presence(strided, 5), obg.build_presence(dev, 5))
    m2 = obg.build_background_model_device(strided, cfg)
    assert m2.trees[0][0] == model.trees[0][0]
    for bad in (dev[..., :2], dev.to(cuda.int16), dev[0]):
        with pytest.raises(ValueError):
            obg.classify(model, bad)
        with pytest.raises(ValueError):
            obg.build_presence(bad, 5)
    truth = cuda.zeros((6, 24, 40), dtype=cuda.uint8)
    st = obg.classify_confusion(model, strided, truth)
    assert st.false_pos == int(want.sum())


@pytest.mark.parametrize("levels", range(1, 9))
def test_counts_histogram_all_levels(cuda, levels):
    """a13 occupancy counts through the histogram kernel (k_hist: shared
    memory at L <= 5, distributed shared memory of a CTA cluster at L = 6,
    global at L >= 7) on flat frames -- a single-colour hot
    spot, uniform-random frames and a noisy gradient, group sizes 1 and 3,
    CTA ranges that split trees -- against np.bincount of the oracle codes."""
    rng = np.random.default_rng(100 + levels)
    h, w = 40, 64
    const = np.empty((3, h, w, 3), np.uint8)
    const[...] = rng.integers(0, 256, size=3, dtype=np.uint8)
    uni = rng.integers(0, 256, size=(4, h, w, 3), dtype=np.uint8)
    grad = np.clip(np.arange(w)[None, None, :, None] * 3 + rng.integers(-9, 10, size=(5, h, w, 3)), 0,
                   255).astype(np.uint8)
    big = rng.integers(0, 256, size=(2, 720, 1280, 3), dtype=np.uint8)
    big[1, :, :640] = (7, 200, 90)
    for frames in (const, uni, grad, big):
        for gs in (1, 3):
            if len(frames) < gs:
                continue
            dev = cuda.from_numpy(frames).cuda()
            pyr, cnt = obg.build_presence(dev, levels, group_size=gs, counts=True)
            ref_pyr = obg.build_presence(dev, levels, group_size=gs)
            assert cuda.equal(pyr, ref_pyr)
            cnt = cnt.cpu().numpy().view(np.uint32)
            for g in range(len(frames) // gs):
                codes = orc.pack_codes(frames[g * gs:(g + 1) * gs], levels).ravel()
                want = np.bincount(codes, minlength=8 ** levels)
                assert np.array_equal(cnt[g, 0], want), (levels, gs, g)


@pytest.mark.parametrize("levels,n_codes", [(6, 200000), (7, 0), (7, 1500000), (8, 3000), (8, 2500000)])
def test_device_serializer_large_trees(cuda, levels, n_codes):
    """obg_serialize (multi-CTA prefix scan) on large trees -- a full depth-7
    cube (2.4 M nodes), millions of random depth-8 codes spanning many scan
    chunks -- against the host sparse serialisation; the device bytes also
    decode back to the same tree."""
    rng = np.random.default_rng(levels * 7 + n_codes)
    host = Octree(levels)
    host._store_codes(np.arange(8 ** levels) if n_codes == 0 else rng.integers(0, 8 ** levels, size=n_codes))
    want = host.to_bytes()
    dev_tree = Octree._from_device(host._device(), levels)
    got = dev_tree.to_bytes()
    assert got == want
    assert Octree.from_bytes(got, levels) == host


@pytest.mark.gpu
@pytest.mark.parametrize("shape,n,levels,grid", [((1, 1), 3, 4, (1, 1)), ((7, 5), 9, 6, (1, 1)), ((48, 64), 5, 5, (2, 3)),
                                                  ((120, 160), 4, 7, (1, 1)), ((33, 17), 2, 8, (1, 1)),
                                                  ((1080, 1920), 2, 6, (1, 1))])
def test_detect_host_matches_device_classify(cuda, shape, n, levels, grid):
    """obg_detect_host (host frames in, host masks out: the reference's
    detect_octree signature, detect.py:22-53) against the device classify and
    the oracle, single frames and batches, odd sizes, grids."""
    import torch
    h, w = shape
    rng = np.random.default_rng(h * 131 + w + levels)
    base = rng.integers(0, 256, size=(1, 1, 1, 3))
    train = np.clip(base + rng.integers(-20, 21, size=(6, h, w, 3)), 0, 255).astype(np.uint8)
    probe = np.clip(base + rng.integers(-40, 41, size=(n, h, w, 3)), 0, 255).astype(np.uint8)
    cfg = obg.ModelConfig(levels=levels, threshold=0.5, grid_rows=grid[0], grid_cols=grid[1], training_frames=6)
    model = obg.build_background_model(list(train), cfg)
    want_dev = obg.classify(model, torch.from_numpy(probe).cuda()).cpu().numpy().astype(bool)
    got_batch = obg.detect_octree_batch(model, probe)
    assert got_batch.dtype == np.bool_ and got_batch.shape == (n, h, w)
    assert np.array_equal(got_batch, want_dev)
    for i in range(n):
        got = obg.detect_octree(model, probe[i])
        assert got.dtype == np.bool_ and np.array_equal(got, want_dev[i])
    # a non-contiguous frame view is accepted like any numpy input
    assert np.array_equal(obg.detect_octree(model, probe[0][:, ::-1][:, ::-1]), want_dev[0])
    if h * w <= 160 * 120:
        trees = orc.build_background_model(list(train), levels, 0.5, grid[0], grid[1])
        assert np.array_equal(got_batch[0], orc.detect_octree(trees, probe[0], levels, grid[0], grid[1]))


@pytest.mark.gpu
def test_detect_host_many_frames_cross_staging_passes(cuda):
    """More frames than one staging pass holds (64 MiB): the passes line up."""
    import torch
    rng = np.random.default_rng(99)
    h, w, n = 540, 960, 60                                      # 1.5 MB per frame: 44 frames per pass
    train = rng.integers(100, 140, size=(4, h, w, 3), dtype=np.uint8)
    probe = rng.integers(90, 150, size=(n, h, w, 3), dtype=np.uint8)
    cfg = obg.ModelConfig(levels=5, threshold=0.5, training_frames=4)
    model = obg.build_background_model(list(train), cfg)
    want = obg.classify(model, torch.from_numpy(probe).cuda()).cpu().numpy().astype(bool)
    assert np.array_equal(obg.detect_octree_batch(model, probe), want)
    # the calling thread's staging buffers can be released and are rebuilt on demand
    _lib.load().obg_host_stage_release()
    assert np.array_equal(obg.detect_octree(model, probe[3]), want[3])
    _lib.load().obg_host_stage_release()


@pytest.mark.gpu
@pytest.mark.parametrize("n_cells,drop", [(300, 0), (300, 1), (0, 0), (4000, 0)])
def test_l7_full_cell_models(cuda, n_cells, drop):
    """L = 7 models whose occupied L=6 cells hold all 8 leaves classify through
    the L=6 kernel on the full-cell bitset (k_l7_states' third operand part);
    dropping one leaf (drop=1) makes a cell partial and must fall back to the
    L=7 kernels.  Checked against the oracle and against a host-side bit test."""
    import torch
    rng = np.random.default_rng(1000 + n_cells + drop)
    h, w = 192, 256
    cells = rng.choice(1 << 18, size=n_cells, replace=False)
    r6, g6, b6 = (cells >> 12) & 63, (cells >> 6) & 63, cells & 63
    leaves = []
    for d in range(8):                                           # all 8 children of each cell
        leaves.append(np.stack([(2 * r6 + (d >> 2)) << 1, (2 * g6 + ((d >> 1) & 1)) << 1, (2 * b6 + (d & 1)) << 1], 1))
    px = np.concatenate(leaves).astype(np.uint8) if n_cells else np.zeros((0, 3), np.uint8)
    if drop and len(px):
        px = px[1:]                                              # one leaf missing: its cell is partial
    frame = np.zeros((h, w, 3), np.uint8)
    flat = frame.reshape(-1, 3)
    if len(px):
        reps = -(-flat.shape[0] // len(px))
        flat[:] = np.tile(px, (reps, 1))[:flat.shape[0]]
    else:
        flat[:] = (1, 1, 1)                                      # a single leaf: one partial cell -> not the cells path
    train = np.stack([frame, frame])
    cfg = obg.ModelConfig(levels=7, threshold=0.5, training_frames=2)
    model = obg.build_background_model(list(train), cfg)
    probe = rng.integers(0, 256, size=(3, h, w, 3), dtype=np.uint8)
    probe[0].reshape(-1, 3)[:len(flat) // 2] = flat[:len(flat) // 2] ^ rng.integers(0, 2, size=(len(flat) // 2, 3), dtype=np.uint8)
    probe[1] = frame
    got = obg.classify(model, torch.from_numpy(probe).cuda()).cpu().numpy().astype(bool)
    # host-side truth: a pixel is background iff its 7-bit colour is a training colour
    key = lambda a: (a[..., 0].astype(np.int64) >> 1) << 14 | (a[..., 1].astype(np.int64) >> 1) << 7 | (a[..., 2].astype(np.int64) >> 1)
    present = np.zeros(1 << 21, bool)
    present[key(flat)] = True
    assert np.array_equal(got, ~present[key(probe)])
    assert not got[1].any()
    trees = orc.build_background_model(list(train), 7, 0.5, 1, 1)
    assert np.array_equal(got[2], orc.detect_octree(trees, probe[2], 7, 1, 1))
    # the same model loaded from its bytes (host tree -> obg_leaf_cube -> k_l7_states)
    loaded = obg.read_model(obg.write_model(model))
    assert np.array_equal(obg.detect_octree_batch(loaded, probe), got)
    # bit-packed output takes the same path
    packed = obg.classify(model, torch.from_numpy(probe).cuda(), packed=True).cpu().numpy()
    assert np.array_equal(np.unpackbits(packed, axis=1, bitorder="little")[:, :h * w].reshape(3, h, w).astype(bool), got)


@pytest.mark.gpu
@pytest.mark.parametrize("level", ["0", "1", "2"])
def test_dependent_launch_levels(cuda, level):
    """OBG_PDL = 0 / 1 / 2 (no programmatic dependent launches / the merge /
    also a classify flagged after_build): the same model and masks, eagerly and
    as a captured step.  The level is read once per process, hence a child."""
    import subprocess
    import sys
    import textwrap
    code = textwrap.dedent('''
        import hashlib, numpy as np, torch
        import paper_1412_1945_b200 as obg
        from paper_1412_1945_b200.pipeline import CapturedStep
        rng = np.random.default_rng(5)
        base = rng.integers(0, 256, size=(1, 1, 1, 3))
        train = torch.from_numpy(np.clip(base + rng.integers(-30, 31, size=(12, 96, 128, 3)), 0, 255).astype(np.uint8)).cuda()
        test = torch.from_numpy(np.clip(base + rng.integers(-60, 61, size=(5, 96, 128, 3)), 0, 255).astype(np.uint8)).cuda()
        h = hashlib.sha256()
        for L in (4, 5, 6):
            cfg = obg.ModelConfig(levels=L, threshold=0.5, training_frames=12)
            m = obg.build_background_model_device(train, cfg)
            masks = obg.classify(m, test, after_build=True)
            step = CapturedStep(train, test, cfg)
            for _ in range(3):
                out = step.step()
            torch.cuda.synchronize()
            assert torch.equal(out, masks)
            assert step.model.trees[0][0].to_bytes() == m.trees[0][0].to_bytes()
            h.update(m.trees[0][0].to_bytes()); h.update(masks.cpu().numpy().tobytes())
        print("DIGEST", h.hexdigest())
    ''')
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for lv in sorted({"0", level}):
        env = dict(os.environ, OBG_PDL=lv, PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""))
        res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
        assert res.returncode == 0, res.stderr[-2000:]
        outs[lv] = [ln for ln in res.stdout.splitlines() if ln.startswith("DIGEST")][0]
    assert outs[level] == outs["0"]
