"""Per-call latency of small integer permanents through the public API (the
reference's default dispatch for int64: combinatoric / Glynn / Ryser with
checked int64), and small float combinatoric calls.

    python tools/small_int_probe.py"""
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03421_b200 as P  # noqa: E402

rng = np.random.default_rng(0)
cases = [("opt int 3x3", P.opt, np.array([[1, 2, 3], [4, 5, 6], [7, 8, 9]])),
         ("opt int 6x6", P.opt, rng.integers(-3, 4, (6, 6))),
         ("opt int 10x10", P.opt, rng.integers(0, 2, (10, 10))),
         ("opt int 14x14", P.opt, rng.integers(0, 2, (14, 14))),
         ("glynn int 12x12", P.glynn, rng.integers(0, 2, (12, 12))),
         ("ryser int 12x12", P.ryser, rng.integers(0, 2, (12, 12))),
         ("combinatoric int 8x8", P.combinatoric, rng.integers(0, 3, (8, 8))),
         ("combinatoric f64 5x5", P.combinatoric, rng.uniform(-1, 1, (5, 5))),
         ("combinatoric f64 4x10", P.combinatoric, rng.uniform(-1, 1, (4, 10))),
         ("opt f64 6x6", P.opt, rng.uniform(-1, 1, (6, 6)))]
for name, fn, a in cases:
    for _ in range(5):
        fn(a)
    ts = []
    for _ in range(200):
        t = time.perf_counter()
        fn(a)
        ts.append(time.perf_counter() - t)
    print(f"{name:24s} {statistics.median(ts) * 1e6:8.1f} us", flush=True)
