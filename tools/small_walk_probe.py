"""Small single permanents (the metric's n = 20..26 end):
per-call latency through the C ABI and the walk kernel's device time.

    python tools/small_walk_probe.py [reps] [n ...]   (n: Glynn sizes only)
Prints, per n: median call time of perm_glynn_f64 on a host matrix (the
public entry point minus Python), the walk kernel's CUDA-event time, the
launch plan, and the fraction of the FP64 pipe the kernel reaches."""
import ctypes as C
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03421_b200 as P  # noqa: E402
from paper_2510_03421_b200 import _lib, workloads as W  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
lib = _lib.load()
lib.perm_set_timing(1)
PEAK = 148 * 64 * 1.965e9
out = _lib.out_buf(2)
plan = (("glynn", range(14, 29)), ("ryser", (20, 24)))
if len(sys.argv) > 2:
    plan = (("glynn", [int(x) for x in sys.argv[2:]]),)
for alg, ns in plan:
    fn = lib.perm_glynn_f64 if alg == "glynn" else lib.perm_ryser_f64
    for n in ns:
        a = W.c5(n)
        ptr = C.c_void_p(a.ctypes.data)
        for _ in range(20):
            fn(n, n, ptr, n, 0, out, None, None)
        ts, ks = [], []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn(n, n, ptr, n, 0, out, None, None)
            ts.append(time.perf_counter() - t0)
            ks.append(lib.perm_last_kernel_ms())
        api = None
        if alg == "glynn":  # the public Python API on the same host matrix
            pf = P.glynn
            for _ in range(10):
                pf(a)
            tp = []
            for _ in range(min(reps, 100)):
                t0 = time.perf_counter()
                pf(a)
                tp.append(time.perf_counter() - t0)
            api = statistics.median(tp)
        g, l2 = C.c_int(), C.c_int()
        lib.perm_last_kernel_plan(C.byref(g), C.byref(l2))
        steps = (1 << (n - 1)) if alg == "glynn" else (1 << n)
        k = statistics.median(ks) * 1e-3
        print(f"{alg} n={n}: call {statistics.median(ts) * 1e6:7.1f} us  "
              f"{'' if api is None else f'P.glynn {api * 1e6:7.1f} us  '}kernel {k * 1e6:7.1f} us  "
              f"grid {g.value:4d} log2L {l2.value:2d}  pipe {steps * 2 * n / k / PEAK:6.1%}  value {out[0]:.6e}",
              flush=True)
