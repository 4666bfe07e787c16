"""Frame ingest: the native PPM / PGM codecs match the
reference's decoded arrays, error messages and byte offsets on every
recorded case, and the threaded sequence reader / mask writer agree with the
per-file codecs.  CPU only (host code in libobg.so)."""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

import paper_1412_1945_b200 as obg
from paper_1412_1945_b200.errors import FormatError

HERE = os.path.dirname(os.path.abspath(__file__))


def _cases():
    sys.path.insert(0, os.path.join(HERE, "golden"))
    saved = sys.modules.get("make_golden")
    sys.modules["make_golden"] = type(sys)("make_golden")     # the case builder needs no reference
    try:
        from make_golden_io import io_cases
        return io_cases()
    finally:
        if saved is not None:
            sys.modules["make_golden"] = saved
        else:
            del sys.modules["make_golden"]


def test_codecs_match_reference():
    with open(os.path.join(HERE, "golden", "golden_io.json")) as f:
        golden = json.load(f)["cases"]
    cases = _cases()
    assert len(cases) == len(golden)
    for (kind, data), rec in zip(cases, golden):
        fn = obg.read_ppm if kind == "ppm" else obg.read_mask_pgm
        try:
            a = fn(data)
            got = {"ok": True, "shape": list(a.shape),
                   "sha": hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()}
        except FormatError as e:
            got = {"ok": False, "type": "FormatError", "msg": str(e), "offset": e.offset}
        want = {k: v for k, v in rec.items() if k != "kind"}
        assert got == want, data[:40]


def test_round_trips_and_writers():
    rng = np.random.default_rng(3)
    f = rng.integers(0, 256, size=(7, 5, 3), dtype=np.uint8)
    assert np.array_equal(obg.read_ppm(obg.write_ppm(f)), f)
    m = rng.random((7, 5)) < 0.5
    assert np.array_equal(obg.read_mask_pgm(obg.write_mask_pgm(m)), m)
    with pytest.raises(ValueError, match="expected"):
        obg.write_ppm(f[..., :2])
    with pytest.raises(ValueError, match="expected"):
        obg.write_mask_pgm(m.astype(np.uint8))


def test_sequence_batch_reader(tmp_path):
    rng = np.random.default_rng(4)
    frames = rng.integers(0, 256, size=(9, 33, 47, 3), dtype=np.uint8)
    seq = obg.write_frame_sequence(tmp_path / "seq", list(frames))
    assert len(seq) == 9 and (seq.width, seq.height) == (47, 33)
    # a long header comment (header beyond the reader's first block)
    (tmp_path / "seq" / seq.names[4]).write_bytes(b"P6\n#" + b"x" * 6000 + b"\n47 33\n255\n" + frames[4].tobytes())
    assert np.array_equal(np.stack(seq.load_all()), frames)
    for threads in (1, 3, 0):
        got = seq.load_batch(pinned=False, threads=threads)
        assert np.array_equal(got, frames)
    assert np.array_equal(seq.load_batch([8, 0, 3], pinned=False), frames[[8, 0, 3]])
    # errors: truncated file (FormatError with the reference's offset), size mismatch (ValueError)
    p = tmp_path / "seq" / seq.names[2]
    p.write_bytes(obg.write_ppm(frames[2])[:-5])
    with pytest.raises(FormatError, match="truncated pixel data") as ei:
        seq.load_batch(pinned=False)
    assert ei.value.offset == len(b"P6\n47 33\n255\n")
    p.write_bytes(obg.write_ppm(frames[2][:, :40]))
    with pytest.raises(ValueError, match=f"frame {seq.names[2]} is 40x33, sequence is 47x33"):
        seq.load_batch(pinned=False)
    with pytest.raises(ValueError, match="no .ppm frames"):
        obg.FrameSequence.scan(tmp_path / "empty_dir_that_does_not_exist")


def test_mask_writer(tmp_path):
    rng = np.random.default_rng(5)
    masks = rng.random((6, 19, 23)) < 0.4
    paths = [tmp_path / f"m{i}.pgm" for i in range(6)]
    obg.save_masks(masks, paths, threads=3)
    for m, p in zip(masks, paths):
        assert p.read_bytes() == obg.write_mask_pgm(m)
    obg.save_masks(masks.astype(np.uint8) * 7, paths)          # any nonzero byte is foreground
    assert all(np.array_equal(obg.load_mask(p), m) for m, p in zip(masks, paths))


@pytest.mark.gpu
def test_detect_sequence_pipeline(cuda, tmp_path):
    """PPM directory -> model + masks through the ingest pipeline equals the
    in-memory path and the oracle; masks written as PGM files match too."""
    from oracle import octree_oracle as orc
    from paper_1412_1945_b200 import pipeline, scenes
    sc = scenes.generate(0)
    frames = np.concatenate([sc.train, sc.test])
    seq = obg.write_frame_sequence(tmp_path / "frames", list(frames))
    cfg = obg.ModelConfig(levels=sc.config.levels, threshold=sc.config.threshold, training_frames=len(sc.train))
    model, masks = pipeline.detect_sequence(seq, cfg, batch=7, chunk=3)
    want_model = orc.build_background_model(list(sc.train), cfg.levels, cfg.threshold)
    assert model.trees[0][0].to_bytes() == orc.to_bytes(want_model[(0, 0)])
    want = np.stack([orc.detect_octree(want_model, f, cfg.levels) for f in frames])
    assert np.array_equal(masks.numpy().astype(bool), want)
    model2, none = pipeline.detect_sequence(tmp_path / "frames", cfg, out_dir=tmp_path / "masks", batch=8)
    assert none is None
    for i, name in enumerate(seq.names):
        assert np.array_equal(obg.load_mask(tmp_path / "masks" / name.replace(".ppm", ".pgm")), want[i])
