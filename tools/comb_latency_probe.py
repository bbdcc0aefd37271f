"""Single float combinatoric latency (public API) over small shapes, to place
the tiny-path threshold PERM_TINY_COMB_MAX_M (batch-of-one thread DFS through
mapped memory) against the tree-split comb kernel.

    PERM_TINY_COMB_MAX_M=4|8 python tools/comb_latency_probe.py"""
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03421_b200 as P  # noqa: E402

rng = np.random.default_rng(0)
for m, n in ((4, 4), (5, 5), (6, 6), (7, 7), (8, 8), (5, 8), (5, 10), (6, 9), (6, 12), (7, 10)):
    a = rng.uniform(-1, 1, (m, n))
    for _ in range(3):
        P.combinatoric(a)
    ts = []
    for _ in range(51):
        t = time.perf_counter()
        P.combinatoric(a)
        ts.append(time.perf_counter() - t)
    print(f"{m}x{n}: {statistics.median(ts) * 1e6:8.1f} us", flush=True)
