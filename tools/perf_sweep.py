"""Per-config timings on the GPU (all BASELINE.json configs + the n-sweep),
written as JSON for profiles/.  Kernel-level numbers come from CUDA events
around the C-ABI calls on the launching stream (synchronizing calls), e2e
numbers from the public API with host inputs.

    python tools/perf_sweep.py gpurun_out/perf_r1.json
"""
from __future__ import annotations

import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2510_03421_b200 as P  # noqa: E402
from paper_2510_03421_b200 import _lib, workloads as W  # noqa: E402

PEAK = None


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return statistics.median(ts)


def kernel_ms():
    return _lib.load().perm_last_kernel_ms()


def main(out):
    lib = _lib.load()
    lib.perm_set_timing(1)
    pk = _lib.out_buf(1)
    _lib.check(lib.perm_fp64_pipe_probe(0, 0.5, pk), "probe")
    dfma = float(pk[0])
    _lib.check(lib.perm_fp64_pipe_probe(1, 0.5, pk), "probe")
    peak = max(dfma, float(pk[0]))  # DADD/DMUL chains reach the nominal rate; DFMA ~8% less
    res = {"fp64_probe_dfma_per_s": dfma, "fp64_probe_dadd_dmul_per_s": float(pk[0]),
           "frac_peak_denominator": peak, "configs": {}}
    R = res["configs"]

    # C5 n-sweep (Glynn f64, U[0,1]/n) and Ryser f64 for comparison
    for n in list(range(20, 37, 2)):
        a = W.c5(n)
        t = timeit(lambda: P.glynn(a), reps=3 if n >= 34 else 5)
        km = kernel_ms()
        steps = 2 ** (n - 1)
        R[f"glynn_f64_n{n}"] = {"e2e_s": t, "kernel_ms": km, "steps_per_s_kernel": steps / (km * 1e-3),
                                "frac_peak": steps * 2 * n / (km * 1e-3) / peak}
        if n <= 32:
            t = timeit(lambda: P.ryser(a), reps=3)
            km = kernel_ms()
            R[f"ryser_f64_n{n}"] = {"e2e_s": t, "kernel_ms": km, "subsets_per_s_kernel": 2 ** n / (km * 1e-3),
                                    "frac_peak": 2 ** n * 2 * n / (km * 1e-3) / peak}
    # C3a / C3b
    for name, a in (("c3a_glynn_c128_24x24", W.c3a()), ("c3b_glynn_c128_20x28", W.c3b())):
        m, n = a.shape
        t = timeit(lambda: P.glynn(a))
        km = kernel_ms()
        steps = 2 ** (n - 1)
        R[name] = {"e2e_s": t, "kernel_ms": km, "steps_per_s_kernel": steps / (km * 1e-3),
                   "frac_peak": steps * (6 * n - 2) / (km * 1e-3) / peak}
    b = W.c3b()
    t = timeit(lambda: P.ryser(b), reps=3)
    km = kernel_ms()
    R["c3b_ryser_c128_20x28"] = {"e2e_s": t, "kernel_ms": km}
    # C4 exact int128 and checked
    for name, a in (("c4a_01_n32", W.c4a()), ("c4b_pm2_n28", W.c4b())):
        n = a.shape[0]
        t = timeit(lambda: P.glynn(a, exact="int128"), reps=3, warm=1)
        R[f"{name}_glynn_int128"] = {"e2e_s": t, "steps_per_s_e2e": 2 ** (n - 1) / t,
                                     "note": "includes the FP64 certificate walk"}
        t = timeit(lambda: P.ryser(a, exact="int128"), reps=3, warm=1)
        R[f"{name}_ryser_int128"] = {"e2e_s": t, "subsets_per_s_e2e": 2 ** n / t}
    # C1: 64 x 12x12 one call each, and as a batch
    A = W.c1()
    t = timeit(lambda: [P.glynn(x) for x in A], reps=3)
    R["c1_glynn_64x12x12_loop"] = {"e2e_s": t, "per_matrix_us": t / 64 * 1e6}
    t = timeit(lambda: P.glynn_batch(A), reps=5)
    R["c1_glynn_64x12x12_batch"] = {"e2e_s": t}
    # C2 batches: host numpy (e2e) and device-resident (kernel)
    import torch

    for name, A in (("c2a_8x8", W.c2a()), ("c2b_4x10", W.c2b())):
        t = timeit(lambda: P.opt_batch(A), reps=3, warm=1)
        dA = torch.tensor(A, device="cuda")
        P.opt_batch(dA)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            P.opt_batch(dA)
        e1.record()
        torch.cuda.synchronize()
        km = e0.elapsed_time(e1) / 10
        R[name] = {"e2e_s": t, "matrices_per_s_e2e": A.shape[0] / t, "device_ms": km,
                   "matrices_per_s_device": A.shape[0] / (km * 1e-3),
                   "hbm_gbs_device": A.nbytes / (km * 1e-3) / 1e9}
    # combinatoric
    for m, n in ((8, 8), (10, 10), (12, 12), (4, 12), (6, 10)):
        a = np.random.default_rng(1).uniform(-1, 1, (m, n))
        t = timeit(lambda: P.combinatoric(a), reps=3, warm=1)
        R[f"comb_f64_{m}x{n}"] = {"e2e_s": t}
    Path(out).write_text(json.dumps(res, indent=1))
    for k, v in R.items():
        print(k, {kk: (f"{vv:.4g}" if isinstance(vv, float) else vv) for kk, vv in v.items()})


if __name__ == "__main__":
    main(sys.argv[1])
