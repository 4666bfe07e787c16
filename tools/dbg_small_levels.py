import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1412_1945_b200 as obg
from oracle import octree_oracle as orc
rng = np.random.default_rng(0)
for L in (1, 2, 3, 4, 5, 6):
    for (n, h, w, gs) in [(1, 4, 4, 1), (2, 4, 4, 1), (2, 4, 4, 2), (5, 8, 2, 1), (3, 16, 16, 1)]:
        f = rng.integers(0, 256, size=(n, h, w, 3), dtype=np.uint8)
        dev = torch.from_numpy(f).cuda()
        pyr = obg.build_presence(dev, L, group_size=gs)
        bad = []
        for g in range(n // gs):
            t = obg.Octree._from_device(pyr[g, 0], L)
            want = orc.build_frame_tree(list(f[g*gs:(g+1)*gs]), (0, 0), L, 1, 1)
            if t.to_bytes() != orc.to_bytes(want):
                bad.append((g, t.leaf_codes()[:10], want.leaf_codes()[:10]))
        print(L, (n, h, w, gs), 'OK' if not bad else bad)
