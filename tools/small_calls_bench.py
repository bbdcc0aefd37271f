"""Per-call latency of small single permanents through each algorithm and opt (zero-copy path)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2510_03421_b200 as P
rng = np.random.default_rng(0)
for (m, n) in ((2, 7), (3, 3), (4, 6), (5, 5), (6, 6), (4, 10), (8, 8), (3, 9), (7, 9)):
    a = rng.uniform(-1, 1, (m, n))
    row = []
    for fn in (P.combinatoric, P.ryser, P.glynn, P.opt):
        fn(a); fn(a)
        t = time.perf_counter()
        for _ in range(200): fn(a)
        row.append((time.perf_counter() - t) / 200 * 1e6)
    print(f"{m}x{n}: comb {row[0]:.1f}  ryser {row[1]:.1f}  glynn {row[2]:.1f}  opt {row[3]:.1f} us", flush=True)
