"""Single square Glynn n = 8..16 per-call latency vs PERM_TINY_GLYNN_MAX_N -> profiles/r1_tiny_glynn_threshold.txt."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2510_03421_b200 as P
rng = np.random.default_rng(0)
for n in range(8, 17):
    a = rng.uniform(-1, 1, (n, n)); c = a + 1j * rng.uniform(-1, 1, (n, n))
    row = []
    for x in (a, c):
        P.glynn(x); P.glynn(x)
        t = time.perf_counter()
        for _ in range(200): P.glynn(x)
        row.append((time.perf_counter() - t) / 200 * 1e6)
    print(f"n={n}: glynn f64 {row[0]:.1f} us  c128 {row[1]:.1f} us", flush=True)
