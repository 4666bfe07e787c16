"""Generate tests/golden/golden.json by running the REFERENCE implementation.

Run in the build container (where the reference is importable):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The reference package is imported from $OCTABG_REF_PATH, else
/root/reference/pkg/src, else baseline/_ref.  Nothing here is needed at test
time: the tests regenerate the (seeded) inputs, check them against the stored
input digests, and compare the oracle / the GPU path with the reference
outputs recorded here.  Large outputs are stored as sha256 digests.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)


def _import_reference():
    for path in (os.environ.get("OCTABG_REF_PATH"), "/root/reference/pkg/src", os.path.join(REPO, "baseline/_ref")):
        if path and os.path.isdir(os.path.join(path, "octabg")):
            sys.path.insert(0, path)
            import octabg
            return octabg
    raise SystemExit("reference package octabg not found")


ref = _import_reference()


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


def mask_digest(mask: np.ndarray) -> str:
    return sha(np.packbits(mask.astype(bool).ravel(), bitorder="little"))


# ---------------------------------------------------------------------------
# small random cases (grids, groups, dead-ends, thresholds)
# ---------------------------------------------------------------------------
from cases import THRESHOLDS, random_case_inputs  # noqa: E402


def random_case_record(case: int) -> dict:
    x = random_case_inputs(case)
    cfg = ref.ModelConfig(levels=x["levels"], threshold=x["threshold"], grid_rows=x["grid_rows"],
                          grid_cols=x["grid_cols"], group_size=x["group_size"],
                          training_frames=len(x["frames"]))
    frames = list(x["frames"])
    model = ref.build_background_model(frames, cfg)
    n_groups = len(frames) // cfg.group_size
    gs = cfg.group_size
    group_trees = [[[ref.build_frame_tree(frames[g * gs:(g + 1) * gs], (r, c), cfg).to_bytes().hex()
                     for c in range(cfg.grid_cols)] for r in range(cfg.grid_rows)] for g in range(n_groups)]
    merged = [[model.trees[r][c].to_bytes().hex() for c in range(cfg.grid_cols)] for r in range(cfg.grid_rows)]
    pruned = {}
    t = model.trees[0][0]
    for nd in range(1, cfg.levels + 1):
        pruned[nd] = t.prune(nd).to_bytes().hex()
    masks = [np.packbits(ref.detect_octree(model, p).ravel(), bitorder="little").tobytes().hex()
             for p in x["probes"]]
    counts0 = np.bincount(ref.pack_codes(x["frames"][0], cfg.levels).ravel(), minlength=8 ** cfg.levels)
    return dict(case=case, levels=cfg.levels, group_size=cfg.group_size, grid_rows=cfg.grid_rows,
                grid_cols=cfg.grid_cols, threshold=cfg.threshold, frames_sha=sha(x["frames"]),
                probes_sha=sha(x["probes"]), group_trees=group_trees, merged=merged, pruned00=pruned,
                masks=masks, counts0_sha=sha(counts0.astype(np.int64)),
                model_file=ref.write_model(model).hex())


# ---------------------------------------------------------------------------
# the five BASELINE configs
# ---------------------------------------------------------------------------
CONFIG_JOBS = [(0, None, "natural"), (1, None, "natural"), (2, None, "natural"), (3, None, "natural")] + \
    [(4, L, v) for v in ("constant", "uniform") for L in (4, 5, 6, 7)]


# Extra records appended by ``--extra`` (without regenerating the rest): C4
# uniform at L7 with threshold 1.0 keeps a leaf only if all 32 training frames
# hit it -- about half of the 2^21 leaves (each frame hits a leaf with
# p = 1 - e^-3.96) -- so the merged tree is partial and the 4K test masks are
# about half foreground: the L7 partial-cell / leaf-mode classify paths are
# pinned (the thr-0.5 uniform records merge to the full cube, masks all 0).
EXTRA_JOBS = [(4, 7, "uniform", 1.0)]


def config_record(job) -> dict:
    from paper_1412_1945_b200 import scenes
    cid, levels, variant = job[:3]
    t0 = time.time()
    sc = scenes.generate(cid, levels=levels, variant=variant)
    threshold = job[3] if len(job) > 3 else sc.config.threshold
    cfg = ref.ModelConfig(levels=sc.config.levels, threshold=threshold,
                          training_frames=len(sc.train))
    train = list(sc.train)
    model = ref.build_background_model(train, cfg)
    tree = model.trees[0][0]
    blob = tree.to_bytes()
    first = [ref.build_frame_tree([train[i]], (0, 0), cfg) for i in range(min(4, len(train)))]
    mask_sha, mask_fg = [], []
    for f in sc.test:
        m = ref.detect_octree(model, f)
        mask_sha.append(mask_digest(m))
        mask_fg.append(int(m.sum()))
    rec = dict(config=cid, variant=variant, levels=cfg.levels, threshold=cfg.threshold,
               width=sc.width, height=sc.height, n_train=len(sc.train), n_test=len(sc.test),
               train_sha=sha(sc.train), test_sha=sha(sc.test),
               merged_sha=sha(blob), merged_len=len(blob), merged_nodes=tree.node_count,
               merged_leaves=len(tree.leaf_codes()),
               merged_hex=blob.hex() if len(blob) <= 65536 else None,
               frame_trees=[dict(sha=sha(t.to_bytes()), leaves=len(t.leaf_codes()),
                                 leaf_sha=sha(np.asarray(t.leaf_codes(), dtype=np.int64))) for t in first],
               counts0_sha=sha(np.bincount(ref.pack_codes(sc.train[0], cfg.levels).ravel(),
                                           minlength=8 ** cfg.levels).astype(np.int64)),
               mask_sha=mask_sha, mask_fg=mask_fg,
               seconds=round(time.time() - t0, 1))
    print(f"config {job}: {rec['seconds']} s, merged {len(blob)} B, fg={sum(mask_fg)}", flush=True)
    return rec


def kat_record() -> dict:
    rng = np.random.default_rng(7)
    px = rng.integers(0, 256, size=(13, 9, 3), dtype=np.uint8)
    kat = dict(
        child_index_200_100_50=[ref.child_index((200, 100, 50), b) for b in range(7, -1, -1)],
        pack_codes_13x9={str(L): ref.pack_codes(px, L).ravel().tolist() for L in (1, 4, 8)},
        pack_codes_13x9_sha=sha(px),
    )
    t = ref.Octree(2)
    t.store((255, 255, 255))
    kat["store_white_d2_bytes"] = t.to_bytes().hex()
    t = ref.Octree(2)
    t.store((0, 0, 0))
    t.store((255, 255, 255))
    kat["store_bw_d2"] = dict(nodes=t.node_count, leaves=t.leaf_codes(), bytes=t.to_bytes().hex())
    t = ref.Octree(4)
    t.store((192, 96, 48))
    kat["prune_4_to_2_leaf_colors"] = sorted(t.prune(2).leaf_colors())
    # merge test vectors of tests/test_model.py:111-120
    def tree_of(colors, levels):
        tr = ref.Octree(levels)
        for c in colors:
            tr.store(c)
        return tr
    trees = [tree_of([(10, 20, 30)], 3), tree_of([(10, 20, 30)], 3), tree_of([(250, 10, 10)], 3)]
    kat["two_of_three"] = {str(th): ref.merge_trees(trees, th, 3).to_bytes().hex() for th in (0.5, 0.7)}
    trees = [tree_of([(0, 0, 0)], 2), ref.Octree(2), ref.Octree(2), ref.Octree(2)]
    kat["empty_in_denominator"] = {str(th): ref.merge_trees(trees, th, 2).to_bytes().hex() for th in (0.25, 0.26)}
    # k_min pins: reference keep decision for count k of total n
    kat["k_min"] = {f"{n}:{th}": min(k for k in range(1, n + 1) if k / n >= th)
                    for n in (1, 2, 3, 7, 10, 20, 30, 50, 64, 100, 255, 512)
                    for th in (0.01, 0.1, 0.25, 0.3, 0.33, 0.5, 0.55, 0.57, 0.58, 0.7, 0.9, 0.99, 1.0)}
    return kat


def main_extra():
    """Append (or replace) the EXTRA_JOBS records in the existing golden.json."""
    path = os.path.join(HERE, "golden.json")
    with open(path) as f:
        out = json.load(f)
    for job in EXTRA_JOBS:
        rec = config_record(job)
        rec["extra"] = True
        out["configs"] = [r for r in out["configs"]
                          if not (r["config"] == rec["config"] and r["variant"] == rec["variant"]
                                  and r["levels"] == rec["levels"] and r["threshold"] == rec["threshold"])]
        out["configs"].append(rec)
    with open(path, "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print(f"updated {path}")


def main():
    if "--extra" in sys.argv:
        return main_extra()
    t0 = time.time()
    out = dict(generator="tests/golden/make_golden.py", reference=getattr(ref, "__version__", "?"),
               numpy=np.__version__)
    out["kat"] = kat_record()
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as pool:
        out["random_cases"] = list(pool.map(random_case_record, range(96)))
    # the 4K stress jobs hold ~4 GB of frames each
    with ProcessPoolExecutor(max_workers=4) as pool:
        out["configs"] = list(pool.map(config_record, CONFIG_JOBS + EXTRA_JOBS))
    path = os.path.join(HERE, "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes) in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
