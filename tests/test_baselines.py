"""Comparison baselines (reference detect.py:56-83):
frame difference and the running mean.  CPU tests pin the oracle to the
reference's recorded outputs (tests/golden/golden_baselines.json, made by
tests/golden/make_golden_baselines.py) and check the host validation; GPU
tests run the CUDA kernels (obg_frame_diff / obg_running_average through the
C ABI) against the same records -- masks bit for bit, running means as the
exact float64 bytes."""

import json
import os

import numpy as np
import pytest

import paper_1412_1945_b200 as obg
from make_golden_baselines import N_CASES, baseline_inputs, sha_f64, sha_mask
from oracle import octree_oracle as orc

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_baselines.json")


@pytest.fixture(scope="module")
def gb():
    with open(GOLDEN) as f:
        return json.load(f)


# ---- CPU: oracle pinned to the reference ------------------------------------------
@pytest.mark.parametrize("case", range(N_CASES))
def test_oracle_baselines(gb, case):
    rec = gb["cases"][case]
    frames, thr, seen = baseline_inputs(case)
    assert list(frames.shape) == rec["shape"] and thr == rec["threshold"] and seen == rec["frames_seen"]
    for t in range(1, len(frames)):
        assert sha_mask(orc.detect_frame_diff(frames[t - 1], frames[t], thr)) == rec["frame_diff"][t - 1]
    avg = frames[0].astype(np.float64)
    s = seen
    for t in range(1, len(frames)):
        m, avg = orc.detect_running_average(s, avg, frames[t], thr)
        s += 1
        assert sha_mask(m) == rec["running_masks"][t - 1]
        assert sha_f64(avg) == rec["running_means"][t - 1]


def test_oracle_bimodal_kat(gb):
    lo = np.zeros((4, 4, 3), np.uint8)
    hi = np.full((4, 4, 3), 255, np.uint8)
    avg = lo.astype(np.float64)
    seen = 1
    for t in range(1, 40):
        _, avg = orc.detect_running_average(seen, avg, hi if t % 2 else lo, 100)
        seen += 1
    assert float(avg[0, 0, 0]) == gb["kat"]["bimodal_mean_after_39"]
    assert abs(float(avg[0, 0, 0]) - 127.5) < 1e-9


def test_validation_messages_without_gpu():
    a = np.zeros((3, 3, 3), np.uint8)
    b = np.zeros((3, 4, 3), np.uint8)
    with pytest.raises(ValueError, match=r"frame difference: dimensions \(3, 3\) vs \(3, 4\) do not match"):
        obg.detect_frame_diff(a, b)
    with pytest.raises(ValueError, match=r"running average: dimensions \(3, 3\) vs \(3, 4\) do not match"):
        obg.detect_running_average(1, a.astype(np.float64), b)
    with pytest.raises(ValueError, match="uint8"):
        obg.detect_frame_diff(a.astype(np.int16), a.astype(np.int16))


# ---- GPU: the CUDA kernels ------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("case", range(N_CASES))
def test_frame_diff_sequence(cuda, gb, case):
    rec = gb["cases"][case]
    frames, thr, _ = baseline_inputs(case)
    masks = obg.frame_diff_sequence(cuda.from_numpy(frames).cuda(), thr).cpu().numpy()
    assert set(np.unique(masks).tolist()) <= {0, 1}
    for t in range(1, len(frames)):
        assert sha_mask(masks[t - 1]) == rec["frame_diff"][t - 1], f"pair {t}"


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(0, N_CASES, 5))
def test_detect_frame_diff_pairs(cuda, gb, case):
    rec = gb["cases"][case]
    frames, thr, _ = baseline_inputs(case)
    for t in range(1, len(frames)):
        m = obg.detect_frame_diff(frames[t - 1], frames[t], thr)
        assert m.dtype == np.bool_ and m.shape == frames.shape[1:3]
        assert sha_mask(m) == rec["frame_diff"][t - 1]


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(N_CASES))
def test_running_average_sequence(cuda, gb, case):
    """One launch over the whole sequence: every mask and the final mean."""
    rec = gb["cases"][case]
    frames, thr, seen = baseline_inputs(case)
    avg = cuda.from_numpy(frames[0].astype(np.float64)).cuda()
    masks = obg.running_average_sequence(cuda.from_numpy(frames[1:].copy()).cuda(), avg, seen, thr).cpu().numpy()
    for t in range(1, len(frames)):
        assert sha_mask(masks[t - 1]) == rec["running_masks"][t - 1], f"frame {t}"
    assert sha_f64(avg.cpu().numpy()) == rec["running_means"][-1]


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(1, N_CASES, 7))
def test_detect_running_average_steps(cuda, gb, case):
    """The reference's one-frame signature, every intermediate mean exact."""
    rec = gb["cases"][case]
    frames, thr, seen = baseline_inputs(case)
    avg = frames[0].astype(np.float64)
    for t in range(1, len(frames)):
        m, avg = obg.detect_running_average(seen + t - 1, avg, frames[t], thr)
        assert sha_mask(m) == rec["running_masks"][t - 1]
        assert sha_f64(avg) == rec["running_means"][t - 1]


@pytest.mark.gpu
def test_bimodal_kat_gpu(cuda, gb):
    lo = np.zeros((4, 4, 3), np.uint8)
    hi = np.full((4, 4, 3), 255, np.uint8)
    seq = np.stack([hi if t % 2 else lo for t in range(1, 40)])
    avg = cuda.from_numpy(lo.astype(np.float64)).cuda()
    masks = obg.running_average_sequence(cuda.from_numpy(seq).cuda(), avg, 1, 100).cpu().numpy()
    assert float(avg[0, 0, 0]) == gb["kat"]["bimodal_mean_after_39"]
    assert masks[10:].all()


@pytest.mark.gpu
def test_baselines_full_size(cuda):
    """1920x1080 sequences (the C3 frame shape): sequence kernels against
    the oracle on sampled frames, the generic (odd-size) path on 1919 columns,
    and the running mean's exactness over 32 frames."""
    from paper_1412_1945_b200 import scenes
    sc = scenes.generate(3, n_train=12, n_test=0)
    frames = sc.train
    dev = cuda.from_numpy(frames).cuda()
    masks = obg.frame_diff_sequence(dev, 30).cpu().numpy()
    for t in (1, 5, 11):
        assert np.array_equal(masks[t - 1].astype(bool), orc.detect_frame_diff(frames[t - 1], frames[t], 30))
    odd = np.ascontiguousarray(frames[:4, :, :1919])
    m2 = obg.frame_diff_sequence(cuda.from_numpy(odd).cuda(), 12).cpu().numpy()
    for t in range(1, 4):
        assert np.array_equal(m2[t - 1].astype(bool), orc.detect_frame_diff(odd[t - 1], odd[t], 12))
    avg_np = frames[0].astype(np.float64)
    avg = cuda.from_numpy(avg_np.copy()).cuda()
    rm = obg.running_average_sequence(dev[1:], avg, 1, 30).cpu().numpy()
    s = 1
    for t in range(1, len(frames)):
        m, avg_np = orc.detect_running_average(s, avg_np, frames[t], 30)
        s += 1
        assert np.array_equal(rm[t - 1].astype(bool), m)
    assert np.array_equal(avg.cpu().numpy().view(np.uint64), avg_np.view(np.uint64))
