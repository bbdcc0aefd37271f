"""FP32-quad exact int128 walk against the FP64-exact walk and the oracle.

gpurun -- python tools/int_f32_probe.py   (PERM_INT_F32=0 selects the FP64-exact walk)
Runs each case in a subprocess per setting so the env switch is read fresh.
"""
import json, os, subprocess, sys, time, statistics
sys.path.insert(0, '.')

CHILD = r'''
import sys, time, statistics, json
sys.path.insert(0, '.')
import numpy as np
import paper_2510_03421_b200 as P
from paper_2510_03421_b200 import workloads as W
from oracle import oracle as O
out = {}
rng = np.random.default_rng(7)
# small cases against the oracle's exact int128 (every quad count 3..8, odd and even)
bad = 0
for n in (9, 10, 12, 13, 14, 16, 17, 18):
    for kind in ("01", "pm2", "pm9"):
        if kind == "01": x = rng.integers(0, 2, (n, n)).astype(np.int64)
        elif kind == "pm2": x = rng.integers(-2, 3, (n, n)).astype(np.int64)
        else: x = rng.integers(-9, 10, (n, n)).astype(np.int64)
        for alg in ("glynn", "ryser"):
            v = getattr(P, alg)(x, exact="int128")
            r = O.exact_int128(alg, x)
            if v != r:
                bad += 1
                print("MISMATCH", n, kind, alg, v, r)
out["small_mismatches"] = bad
fix = json.load(open("tests/golden/c4_exact.json")) if __import__("os").path.exists("tests/golden/c4_exact.json") else None
for name, x in (("c4a", W.c4a()), ("c4b", W.c4b())):
    for alg in ("glynn", "ryser"):
        fn = getattr(P, alg)
        fn(x, exact="int128")
        ts = []
        for _ in range(5):
            t = time.perf_counter(); v = fn(x, exact="int128"); ts.append(time.perf_counter() - t)
        out[f"{name}_{alg}_ms"] = round(statistics.median(ts) * 1e3, 3)
        out[f"{name}_{alg}_value"] = str(v)
print("RESULT " + json.dumps(out))
'''
res = {}
for flag in ("0", "1"):
    env = dict(os.environ, PERM_INT_F32=flag)
    p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    for line in p.stdout.splitlines():
        if line.startswith("RESULT "):
            res[flag] = json.loads(line[7:])
        else:
            print(f"[F32={flag}]", line)
    if p.returncode:
        print(f"[F32={flag}] rc={p.returncode}", p.stderr[-2000:])
for k in sorted(res.get("1", {})):
    print(f"{k:24s} fp64-exact {res.get('0', {}).get(k)}   fp32-quad {res['1'][k]}")
