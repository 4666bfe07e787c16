"""Shared-memory bank-conflict model of the streaming kernels' lookups (CPU).

A warp's lookup j touches pixel 16*lane + j of 32 consecutive 16-pixel units.
The shared word of a pixel in the row layout (csrc/obg.cu, Smem<L>) is
R' * ROWW + G' * GW + (B' >> 5 for L = 6); a lookup costs as many wavefronts
as the largest number of distinct words that share a bank.  Prints, per L,
the row strides (ROWW = GW * 2^L + pad) with the fewest wavefronts averaged
over the synthetic scenes C1-C3, and the one-pad-word stride for comparison.

    python tools/banksim.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1412_1945_b200 import scenes  # noqa: E402


def wavefronts(word):
    n = (len(word) // 512) * 512
    w = np.transpose(word[:n].reshape(-1, 32, 16), (0, 2, 1)).reshape(-1, 32)
    total = 0
    for c in range(0, len(w), 20000):
        ww = np.sort(w[c:c + 20000], axis=1)
        uniq = np.concatenate([np.ones((len(ww), 1), bool), ww[:, 1:] != ww[:, :-1]], axis=1)
        cnt = np.zeros((len(ww), 32), np.int64)
        rows = np.repeat(np.arange(len(ww)), 32).reshape(len(ww), 32)
        np.add.at(cnt, (rows[uniq], (ww % 32)[uniq]), 1)
        total += cnt.max(axis=1).sum()
    return total / len(w)


def main():
    frames = {k: scenes.generate(k, n_train=1, n_test=0).train[:1].reshape(-1, 3).astype(np.int64)
              for k in (1, 2, 3)}
    for L in (6, 5, 4):
        s = 8 - L
        gw = 2 if L == 6 else 1
        base = gw << L
        out = []
        for pad in range(1, 33):
            rw = base + pad
            per = []
            for f in frames.values():
                r, g, b = f[:, 0] >> s, f[:, 1] >> s, f[:, 2] >> s
                per.append(wavefronts(r * rw + g * gw + ((b >> 5) if L == 6 else 0)))
            out.append((round(sum(per) / len(per), 3), rw, [round(x, 2) for x in per]))
        one = [o for o in out if o[1] == base + 1]
        out.sort()
        print(f"L={L} best {out[:4]}  pad=1 {one}")


if __name__ == "__main__":
    main()
