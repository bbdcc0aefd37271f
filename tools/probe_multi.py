import time, json, numpy as np, sys
sys.path.insert(0, '.')
import paper_2510_03421_b200 as P
from paper_2510_03421_b200 import workloads as W
def t(label, f):
    t0 = time.perf_counter(); r = f(); print(f"{label}: {time.perf_counter()-t0:.3f}s", flush=True); return r
a = W.c5(26)
t("glynn single", lambda: P.glynn(a))
for devs in ((0,), (0, 0), (0, 0, 0, 0, 0)):
    t(f"multi {devs}", lambda: P.multi_device_permanent(a, devices=devs))
    t(f"multi again {devs}", lambda: P.multi_device_permanent(a, devices=devs))
t("c3a", lambda: P.multi_device_permanent(W.c3a(), devices=(0, 0, 0), mag=True))
t("ryser", lambda: P.multi_device_permanent(W.c5(22), alg="ryser", devices=(0, 0)))
t("c4b", lambda: P.multi_device_permanent(W.c4b(), devices=(0, 0, 0), exact="int128"))
small = np.random.default_rng(2).integers(-2, 3, (12, 12)).astype(np.int64)
t("small", lambda: P.multi_device_permanent(small, devices=(0, 0)))
