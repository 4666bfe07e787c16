"""Exact-arithmetic check of the reciprocal division used by k_running_average
(div_by in obg.cu): q = RN(q0 + r*y), q0 = RN(d*y), r = d - n*q0, y = RN(1/n)
must equal RN(d/n).  Pure Python (fractions), CPU only."""
import random
from fractions import Fraction as F
random.seed(1)
bad = 0; N = 300000
for i in range(N):
    n = random.randint(2, 1 << 20) if i % 3 else random.randint(2, 64)
    if i % 4 == 0:
        d = float(random.randint(-255, 255))
    else:
        avg = random.uniform(0, 255) if i % 4 == 1 else random.randint(0, 255) + random.choice([1e-9, 1e-13, 0.5, 1/3, 2**-40])
        d = float(random.randint(0, 255)) - avg
    y = 1.0 / n
    q0 = d * y
    r = F(d) - F(n) * F(q0)
    if float(r) != r:
        print("r not exact", d, n); bad += 1; continue
    q1 = float(F(float(r)) * F(y) + F(q0))
    if q1 != d / n:
        bad += 1
        if bad < 5: print("mismatch", d, n, q1, d / n)
print("bad", bad, "of", N)
