"""Partition-formula batches of wide rectangles (runtime-n kernel)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2510_03421_b200 as P
rng = np.random.default_rng(0)
for (m, n) in ((3, 30), (4, 40), (5, 50), (6, 62)):
    A = rng.standard_normal((100_000, m, n)) / np.sqrt(n)
    dA = torch.tensor(A, device="cuda")
    P.partition_batch(dA); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): P.partition_batch(dA)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"1e5 x {m}x{n}: {ms:.3f} ms ({A.nbytes / (ms * 1e-3) / 1e9:.0f} GB/s)", flush=True)
