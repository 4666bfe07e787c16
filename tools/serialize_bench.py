"""f1 timing: OBGM model write (preorder serialisation) of a merged model,
host (numpy, sparse levels) vs device (obg_serialize), and decode back.

    python tools/serialize_bench.py [--config 4 --levels 7 --variant uniform --threshold 1.0]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_1945_b200 as obg  # noqa: E402
from paper_1412_1945_b200 import Octree, scenes  # noqa: E402


def best(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--levels", type=int, default=7)
    ap.add_argument("--variant", default="uniform")
    ap.add_argument("--threshold", type=float, default=0.5)
    ap.add_argument("--frames", type=int, default=32)
    a = ap.parse_args()
    sc = scenes.generate(a.config, n_train=a.frames, n_test=0, levels=a.levels, variant=a.variant)
    cfg = obg.ModelConfig(levels=a.levels, threshold=a.threshold, training_frames=a.frames)
    model = obg.build_background_model_device(torch.from_numpy(sc.train).cuda(), cfg)
    dev_tree = model.trees[0][0]
    blob = dev_tree.to_bytes()
    nodes = dev_tree.node_count
    levels = dev_tree._levels()
    host_tree = Octree._from_levels(levels, a.levels, True)

    def dev_write():
        m = obg.BackgroundModel(cfg, model.frame_width, model.frame_height, _device_pyramids=model._dev_pyr,
                                _device_cube=model._dev_cube)
        return obg.write_model(m)

    def host_write():
        host_tree._bytes = None
        return host_tree.to_bytes()

    t_dev = best(dev_write)
    t_host = best(host_write)
    t_dec = best(lambda: Octree.from_bytes(blob, a.levels))
    assert host_write() == blob
    print(json.dumps({"workload": f"C{a.config} {a.variant} L{a.levels} thr{a.threshold} merged tree of {a.frames} frames",
                      "nodes": nodes, "bytes": len(blob),
                      "write_model_device_ms": round(1000 * t_dev, 3), "to_bytes_host_sparse_ms": round(1000 * t_host, 3),
                      "from_bytes_native_ms": round(1000 * t_dec, 3)}))


if __name__ == "__main__":
    main()
