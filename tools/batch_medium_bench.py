"""Batched square Glynn for n = 17..30 (walk_multi_kernel) vs a loop of glynn() calls -> profiles/r1_batch_medium_walks.txt."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2510_03421_b200 as P
rng = np.random.default_rng(0)
for n, B in ((17, 1000), (20, 1000), (20, 10), (24, 100), (24, 1), (28, 10)):
    A = rng.uniform(-1, 1, (B, n, n)) / n
    dA = torch.tensor(A, device="cuda")
    P.glynn_batch(dA); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): P.glynn_batch(dA)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    t = time.perf_counter()
    for i in range(min(B, 50)): P.glynn(A[i])
    loop = (time.perf_counter() - t) / min(B, 50) * B * 1e3
    ops = B * 2 ** (n - 1) * 2 * n
    print(f"n={n} B={B}: batch {ms:.3f} ms ({ops/(ms*1e-3)/1e12:.2f} Tops)  loop of glynn() {loop:.2f} ms", flush=True)
