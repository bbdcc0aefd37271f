import os, sys, time, statistics
sys.path.insert(0, '.')
import paper_2510_03421_b200 as P
from paper_2510_03421_b200 import workloads as W
a, b = W.c4a(), W.c4b()
for x in (a, b):
    P.glynn(x, exact="int128")
for name, x in (("c4a", a), ("c4b", b)):
    for alg in ("glynn", "ryser"):
        fn = getattr(P, alg)
        ts = []
        for _ in range(3):
            t = time.perf_counter(); v = fn(x, exact="int128"); ts.append(time.perf_counter() - t)
        print(os.environ.get("PERMANENT_B200_LIB", "default").split("/")[-1], name, alg, f"{statistics.median(ts)*1e3:.2f} ms", v % 1000)
