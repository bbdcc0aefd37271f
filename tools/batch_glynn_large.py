"""Large batches of square Glynn n = 9..13 (thread- vs warp-per-matrix; PERM_BATCH_WARP_MIN_N) -> profiles/r1_batch_glynn_large.txt."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2510_03421_b200 as P
rng = np.random.default_rng(0)
for n, B in ((9, 200000), (10, 200000), (11, 200000), (12, 200000), (13, 100000)):
    A = rng.uniform(-1, 1, (B, n, n)) / n
    dA = torch.tensor(A, device="cuda")
    P.glynn_batch(dA); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): P.glynn_batch(dA)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{B:.0e} x {n}x{n}: {ms:.3f} ms ({B * 2**(n-1) * 2 * n / (ms*1e-3) / 1e12:.2f} Tops)", flush=True)
