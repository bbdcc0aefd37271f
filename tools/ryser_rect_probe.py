"""Rectangular Ryser: all-subsets weighted Gray walk vs the reference's
combination order, per-call latency through the public API (P.ryser on a host
float64 matrix), to place ryser_rect_use_comb's crossover.

    PERM_RYSER_RECT=walk|comb python tools/ryser_rect_probe.py
"""
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03421_b200 as P  # noqa: E402

rng = np.random.default_rng(0)
for n in (12, 14, 16, 18, 20, 21, 22, 23, 24, 26, 28):
    row = []
    for m in (2, 3, 4, 6, 8):
        if m >= n:
            continue
        a = rng.standard_normal((m, n)) / np.sqrt(n)
        for _ in range(3):
            P.ryser(a)
        reps = 31 if n <= 24 else 5
        ts = []
        for _ in range(reps):
            t = time.perf_counter()
            P.ryser(a)
            ts.append(time.perf_counter() - t)
        row.append(f"{m}x{n} {statistics.median(ts) * 1e6:8.1f}")
    print("  ".join(row), flush=True)
