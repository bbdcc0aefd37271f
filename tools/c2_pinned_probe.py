"""C2a / C2b end to end from pageable numpy vs a pinned torch tensor (the DMA
reads page-locked input in place): gpurun -- python tools/c2_pinned_probe.py"""
import sys, time, statistics
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2510_03421_b200 as P
from paper_2510_03421_b200 import workloads as W
for name, A in (("C2a 1e6x8x8", W.c2a()), ("C2b 1e6x4x10", W.c2b())):
    T = torch.from_numpy(A).pin_memory()
    for label, x in (("pageable numpy", A), ("pinned tensor", T)):
        P.opt_batch(x)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter(); P.opt_batch(x); ts.append(time.perf_counter() - t0)
        ms = statistics.median(ts) * 1e3
        print(f"{name} {label:15s} {ms:7.2f} ms  {A.nbytes / ms / 1e6:6.1f} GB/s")
