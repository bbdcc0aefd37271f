"""Batches of m >= 7 rectangles, n = 10..16: the dispatch (opt_batch) vs explicit Glynn (warp per matrix, ones-padded, pre-scaled) and Ryser -> profiles/r1_batch_rect_mid.txt."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2510_03421_b200 as P
rng = np.random.default_rng(0)
for m, n in ((7, 10), (7, 12), (8, 13), (10, 14), (12, 16), (15, 16)):
    A = rng.uniform(-1, 1, (10000, m, n)) / n
    dA = torch.tensor(A, device="cuda")
    row = []
    for fn in (P.opt_batch, P.glynn_batch, P.ryser_batch):
        fn(dA); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): fn(dA)
        e1.record(); torch.cuda.synchronize()
        row.append(e0.elapsed_time(e1) / 3)
    print(f"1e4 x {m}x{n}: opt {row[0]:.3f} ms  glynn {row[1]:.3f} ms  ryser {row[2]:.3f} ms", flush=True)
