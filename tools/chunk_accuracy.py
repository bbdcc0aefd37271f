"""C5 accuracy and time vs the walk chunk cap (run with PERM_WALK_MAX_LOG2L=8..14) -> DESIGN 2.5 table."""
import os, sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2510_03421_b200 as P
from paper_2510_03421_b200 import workloads as W, engine as E, _lib
a = W.c5(36)
(rh, rl), _ = E.walk_dd("ryser", a)
ref = rh + rl
P.glynn(a)
ts = []
for _ in range(3):
    t = time.perf_counter(); v = P.glynn(a); ts.append(time.perf_counter() - t)
print(os.environ.get("PERM_WALK_MAX_LOG2L", "default"), "rel", abs(v - ref) / abs(ref), "time", min(ts))
for name, A, r in (("J36", np.ones((36, 36)), float(np.prod(np.arange(1, 37, dtype=np.float64))),),):
    vv = P.glynn(A); print(name, "rel", abs(vv - r) / r)
