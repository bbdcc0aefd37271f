"""C2a / C2b host-array e2e time vs copy threads and chunk size (env knobs
PERM_COPY_THREADS / PERM_BATCH_CHUNK_MB are read per call)."""
import os, statistics, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03421_b200 as P
from paper_2510_03421_b200 import workloads as W

A2a, A2b = W.c2a(), W.c2b()
P.opt_batch(A2a[:1000])
for th in (4, 8, 12, 16):
    for ch in (8, 16, 32, 64):
        os.environ["PERM_COPY_THREADS"] = str(th)
        os.environ["PERM_BATCH_CHUNK_MB"] = str(ch)
        for name, A in (("c2a", A2a), ("c2b", A2b)):
            P.opt_batch(A)
            ts = []
            for _ in range(5):
                t = time.perf_counter(); P.opt_batch(A); ts.append(time.perf_counter() - t)
            print(f"threads {th:2d} chunk {ch:3d} MB {name}: {statistics.median(ts)*1e3:.2f} ms", flush=True)
