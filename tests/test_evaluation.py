"""Evaluation: host mirror of the reference's
evaluation.py pinned to its recorded outputs, and the fused device
classify + confusion path (obg_classify_confusion) against the reference's
detect_octree masks and against the host count of our own masks."""

import json
import os

import numpy as np
import pytest

import paper_1412_1945_b200 as obg
from oracle import octree_oracle as orc
from paper_1412_1945_b200 import EvalStats, ModelConfig

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(HERE, "golden", "golden_eval.json")) as f:
        return json.load(f)


def _pairs():
    import sys
    sys.path.insert(0, os.path.join(HERE, "golden"))
    from make_golden_eval import eval_pairs   # seeded inputs only (the reference is not imported at test time)
    return eval_pairs()


def test_host_accumulate_f0_report(gold, monkeypatch):
    import sys
    # make_golden_eval imports the reference through make_golden; stub it so only the seeds are used
    monkeypatch.setitem(sys.modules, "make_golden", type(sys)("make_golden"))
    sys.modules["make_golden"].ref = None
    pairs = _pairs()
    for (p, t), want in zip(pairs, gold["pairs"]):
        s = obg.accumulate(p, t)
        assert [s.true_neg, s.true_pos, s.false_neg, s.false_pos] == want
        assert list(orc.confusion(p, t)) == want
        assert s.total == p.size
    chained = EvalStats()
    for p, t in pairs:
        chained = obg.accumulate(p, t, chained)
    assert [chained.true_neg, chained.true_pos, chained.false_neg, chained.false_pos] == gold["chained"]
    from make_golden_eval import STATS
    for s, want in zip(STATS, gold["f0"]):
        assert list(obg.f0_score(EvalStats(*s))) == want
    assert obg.emit_report([("octree", "c%d" % i, EvalStats(*s)) for i, s in enumerate(STATS)]) == gold["report"]
    with pytest.raises(ValueError, match="mask dimensions"):
        obg.accumulate(np.zeros((2, 2), bool), np.zeros((2, 3), bool))


def _truth(n, h, w, seed):
    return np.random.default_rng(seed).random((n, h, w)) < 0.3


@pytest.mark.gpu
def test_fused_confusion_vs_reference(cuda, gold):
    from paper_1412_1945_b200 import scenes
    for rec in gold["configs"]:
        sc = scenes.generate(rec["config"], n_test=rec["n_test"])
        cfg = ModelConfig(levels=sc.config.levels, threshold=sc.config.threshold, training_frames=len(sc.train))
        model = obg.build_background_model_device(cuda.from_numpy(sc.train).cuda(), cfg)
        truth = _truth(rec["n_test"], sc.height, sc.width, rec["truth_seed"])
        frames = cuda.from_numpy(sc.test).cuda()
        for i, want in enumerate(rec["per_frame"]):
            s = obg.classify_confusion(model, frames[i:i + 1], cuda.from_numpy(truth[i:i + 1]).cuda())
            assert [s.true_neg, s.true_pos, s.false_neg, s.false_pos] == want
        total = obg.classify_confusion(model, frames, cuda.from_numpy(truth).cuda())
        assert [total.true_neg, total.true_pos, total.false_neg, total.false_pos] == \
            [sum(x[k] for x in rec["per_frame"]) for k in range(4)]


@pytest.mark.gpu
def test_fused_confusion_layouts(cuda):
    """u8 0/1, u8 0/255 (PGM values), bool and bit-packed truth; ragged frame
    sizes (tails), grids (generic kernel), every L incl. the L=7 state path;
    counts are added to a given EvalStats."""
    rng = np.random.default_rng(9)
    for levels, (h, w), grid in [(6, (48, 64), (1, 1)), (5, (33, 20), (1, 1)), (4, (30, 50), (2, 3)),
                                 (7, (32, 48), (1, 1)), (3, (16, 16), (1, 1)), (8, (16, 32), (1, 1)),
                                 (6, (7, 9), (1, 1))]:
        base = rng.integers(0, 256, size=(1, 1, 1, 3))
        train = np.clip(base + rng.integers(-20, 21, size=(6, h, w, 3)), 0, 255).astype(np.uint8)
        test = np.clip(base + rng.integers(-40, 41, size=(5, h, w, 3)), 0, 255).astype(np.uint8)
        cfg = ModelConfig(levels=levels, threshold=0.5, grid_rows=grid[0], grid_cols=grid[1], training_frames=6)
        model = obg.build_background_model_device(cuda.from_numpy(train).cuda(), cfg)
        frames = cuda.from_numpy(test).cuda()
        truth = rng.random((5, h, w)) < 0.4
        pred = obg.classify(model, frames).cpu().numpy().astype(bool)
        want = [sum(x) for x in zip(*[orc.confusion(pred[i], truth[i]) for i in range(5)])]
        t_dev = cuda.from_numpy(truth).cuda()
        for t in (t_dev, t_dev.to(cuda.uint8), t_dev.to(cuda.uint8) * 255):
            s = obg.classify_confusion(model, frames, t)
            assert [s.true_neg, s.true_pos, s.false_neg, s.false_pos] == want
        packed = np.packbits(truth.reshape(5, -1), axis=1, bitorder="little")
        s = obg.classify_confusion(model, frames, cuda.from_numpy(packed).cuda(), packed=True)
        assert [s.true_neg, s.true_pos, s.false_neg, s.false_pos] == want
        s2 = obg.classify_confusion(model, frames, t_dev, stats=EvalStats(1, 2, 3, 4))
        assert [s2.true_neg, s2.true_pos, s2.false_neg, s2.false_pos] == [a + b for a, b in zip(want, (1, 2, 3, 4))]
