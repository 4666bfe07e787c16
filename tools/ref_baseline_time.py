import sys, time, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'baseline/_ref')
import octabg
from paper_1412_1945_b200 import scenes
fr = scenes.generate(3, n_train=8, n_test=0).train
t = time.perf_counter()
for i in range(1, 8): octabg.detect_frame_diff(fr[i-1], fr[i], 30)
fd = (time.perf_counter() - t) / 7
avg = fr[0].astype(np.float64); t = time.perf_counter()
for i in range(1, 8): m, avg = octabg.detect_running_average(i, avg, fr[i], 30)
ra = (time.perf_counter() - t) / 7
P = 1920 * 1080
print(f"reference CPU (1 core): frame_diff {fd*1e3:.1f} ms/frame = {P/fd/1e6:.0f} Mpx/s; running_average {ra*1e3:.1f} ms/frame = {P/ra/1e6:.0f} Mpx/s")
