import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_1412_1945_b200 as obg
from paper_1412_1945_b200 import scenes
from paper_1412_1945_b200.pipeline import process_batches
cid = int(sys.argv[1])
sc = scenes.generate(cid)
cfg = sc.config
h_train = torch.from_numpy(sc.train).pin_memory()
h_test = torch.from_numpy(sc.test).pin_memory()
h_masks = torch.empty(sc.test.shape[:3], dtype=torch.uint8).pin_memory()
for chunk in (8, 32, 64):
    for rep in range(6):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        process_batches(h_train, h_test, cfg, out_host=h_masks, chunk=chunk)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        if rep >= 3: print(cid, 'chunk', chunk, 'ms', round((t1 - t0) * 1000, 3))
# pieces
torch.cuda.synchronize(); t0 = time.perf_counter(); d = h_train.cuda(non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
print('h2d train', (t1 - t0) * 1000, 'ms', h_train.numel() / (t1 - t0) / 1e9, 'GB/s')
torch.cuda.synchronize(); t0 = time.perf_counter(); d = h_test.cuda(non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
print('h2d test', (t1 - t0) * 1000, 'ms', h_test.numel() / (t1 - t0) / 1e9, 'GB/s')
m = torch.empty(sc.test.shape[:3], dtype=torch.uint8, device='cuda')
torch.cuda.synchronize(); t0 = time.perf_counter(); h_masks.copy_(m, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
print('d2h masks', (t1 - t0) * 1000, 'ms', m.numel() / (t1 - t0) / 1e9, 'GB/s')
