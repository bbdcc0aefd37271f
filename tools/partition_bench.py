"""Partition-formula batches (m = 4..6) vs the subset-skipping Ryser batch kernel -> profiles/r1_partition_m56.txt."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2510_03421_b200 as P
rng = np.random.default_rng(0)
for (m, n) in ((4, 10), (5, 10), (5, 12), (6, 12), (6, 16), (5, 16)):
    A = rng.standard_normal((1_000_000, m, n)) / np.sqrt(n)
    dA = torch.tensor(A, device="cuda")
    res = {}
    for name, fn in (("partition", P.partition_batch), ("ryser", P.ryser_batch)):
        fn(dA); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): out = fn(dA)
        e1.record(); torch.cuda.synchronize()
        res[name] = (e0.elapsed_time(e1) / 5, out.cpu().numpy())
    err = np.max(np.abs(res["partition"][1] - res["ryser"][1]) / np.maximum(np.abs(res["ryser"][1]), 1e-3))
    print(f"{m}x{n} 1e6: partition {res['partition'][0]:.4f} ms ({A.nbytes/res['partition'][0]/1e6:.0f} GB/s)  ryser {res['ryser'][0]:.4f} ms  maxdiff {err:.1e}", flush=True)
