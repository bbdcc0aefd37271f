"""Generate tests/golden/ fixtures by running the REFERENCE in this container.

TEST INFRASTRUCTURE ONLY.  Imports the reference package from
/root/reference/pkg/src (read-only; numba cache redirected to /tmp) and the
C oracle, and writes small fixtures the GPU box can use without the
reference.  Run:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python oracle/gen_golden.py [--skip-slow]

Outputs (tests/golden/):
  parity.json       the reference's 300 golden vectors
                    (pkg/frontend/tests/fixtures/parity.json), re-serialized
  ref_cases.json    reference outputs (value, overflowed) of every algorithm
                    on seeded int / float / complex matrices, m <= n <= 9,
                    plus the integer-overflow KATs of pkg/tests/test_algorithms.py
  ref_int_walk.json reference int64 results near the overflow onset (0/1 and
                    {-2..2} matrices, n = 10..20)
  c1.npz            config C1 (64 x 12x12) matrices + reference glynn/ryser/opt
  c2_sub.npz        first 512 matrices of C2a / C2b + reference opt and
                    run_algorithm(G, R, C) values
  c3.json           C3a / C3b reference values (+ pre-scaled Glynn-rect) and
                    double-double oracle values
  c4.json           C4a / C4b: reference behaviour (OverflowError) and the
                    exact permanent from the int128 oracle
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
ROOT = Path(__file__).resolve().parents[1]
sys.path = [p for p in sys.path if Path(p or ".").resolve() != Path(__file__).resolve().parent]
sys.path.insert(0, str(ROOT))

import permanent as P  # noqa: E402  (the reference)
from permanent.algorithms import AlgorithmId, run_algorithm  # noqa: E402
from permanent.core import as_matrix  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2510_03421_b200 import workloads as W  # noqa: E402

OUT = ROOT / "tests" / "golden"


def enc(v):
    """JSON-safe encoding of a reference value."""
    if isinstance(v, bool):
        return v
    if isinstance(v, int):
        return {"int": str(v)}
    if isinstance(v, complex):
        return {"re": v.real, "im": v.imag}
    return {"float": float(v)}


def enc_matrix(a: np.ndarray):
    if np.iscomplexobj(a):
        return {"kind": "complex", "re": a.real.tolist(), "im": a.imag.tolist()}
    if a.dtype.kind in "iub":
        return {"kind": "int", "v": [[int(x) for x in row] for row in a]}
    return {"kind": "float", "v": a.tolist()}


def ref_run(a, alg):
    r = run_algorithm(as_matrix(a), alg, compiled=True)
    return enc(r.value), bool(r.overflowed)


def gen_parity():
    src = REF / "frontend" / "tests" / "fixtures" / "parity.json"
    cases = json.loads(src.read_text())
    (OUT / "parity.json").write_text(json.dumps(cases, separators=(",", ":")) + "\n")
    print(f"parity.json: {len(cases)} cases")


def gen_ref_cases():
    g = np.random.default_rng([2510, 3421, 100])
    cases = []
    for n in range(1, 10):
        for m in range(1, n + 1):
            for kind in ("int", "float", "complex"):
                reps = 3 if n <= 7 else 1
                for _ in range(reps):
                    if kind == "int":
                        a = g.integers(-9, 10, (m, n)).astype(np.int64)
                    elif kind == "float":
                        a = g.uniform(-1, 1, (m, n))
                    else:
                        a = g.uniform(-1, 1, (m, n)) + 1j * g.uniform(-1, 1, (m, n))
                    res = {}
                    for alg in AlgorithmId:
                        v, o = ref_run(a, alg)
                        res[alg.value] = {"value": v, "overflowed": o}
                    cases.append({"matrix": enc_matrix(a), "results": res})
    # integer-overflow KATs (pkg/tests/test_algorithms.py:182-209) and edges
    kats = [np.array([[2**62, 3], [5, 2**62]]), np.array([[2**31, 1], [1, 2**31]]),
            np.array([[2**30, 1], [1, 2**30]]), np.array([[2**62, 1], [1, 1]]),
            np.array([[-(2**62), 1, 0], [1, 2**40, 3]]), np.array([[2**61, 2**61], [1, 1]]),
            np.array([[3037000499, 0], [0, 3037000499]]), np.array([[3037000500, 0], [0, 3037000500]])]
    for a in kats:
        a = a.astype(np.int64)
        res = {}
        for alg in AlgorithmId:
            v, o = ref_run(a, alg)
            res[alg.value] = {"value": v, "overflowed": o}
        cases.append({"matrix": enc_matrix(a), "results": res, "kat": True})
    (OUT / "ref_cases.json").write_text(json.dumps(cases, separators=(",", ":")) + "\n")
    print(f"ref_cases.json: {len(cases)} cases")


def gen_ref_int_walk():
    g = np.random.default_rng([2510, 3421, 101])
    cases = []
    for n in range(10, 21):
        for law in ("01", "pm2", "01r"):
            if law == "01":
                a = W.bernoulli01(n, g)
            elif law == "pm2":
                a = g.integers(-2, 3, (n, n)).astype(np.int64)
            else:  # rectangular 0/1
                a = (g.random((max(1, n - 3), n)) < 0.5).astype(np.int64)
            res = {}
            for alg in (AlgorithmId.GLYNN, AlgorithmId.RYSER):
                v, o = ref_run(a, alg)
                res[alg.value] = {"value": v, "overflowed": o}
            exact = O.exact_int128("glynn", a)
            cases.append({"matrix": enc_matrix(a), "results": res, "exact": str(exact)})
    (OUT / "ref_int_walk.json").write_text(json.dumps(cases, separators=(",", ":")) + "\n")
    print(f"ref_int_walk.json: {len(cases)} cases")


def gen_c1():
    A = W.c1()
    g = np.array([P.glynn(a) for a in A])
    r = np.array([P.ryser(a) for a in A])
    o = np.array([P.opt(a) for a in A])
    np.savez_compressed(OUT / "c1.npz", a=A, glynn=g, ryser=r, opt=o)
    print("c1.npz written")


def gen_c2():
    k = 512
    A8 = W.c2a(k)
    A4 = W.c2b(k)
    out = {"a8": A8, "a4": A4}
    for name, A in (("8", A8), ("4", A4)):
        out[f"opt{name}"] = np.array([P.opt(a) for a in A])
        for alg in AlgorithmId:
            out[f"{alg.value[0]}{name}"] = np.array(
                [run_algorithm(as_matrix(a), alg, compiled=True).value for a in A])
        out[f"m{name}"] = np.array([O.glynn_magnitude_sum(a) for a in A])
    np.savez_compressed(OUT / "c2_sub.npz", **out)
    print("c2_sub.npz written")


def gen_c3(skip_slow: bool):
    res = {}
    a = W.c3a()
    t = time.time()
    res["c3a_ref_glynn"] = enc(P.glynn(a))
    res["c3a_ref_ryser"] = enc(P.ryser(a))
    res["c3a_dd_glynn"] = enc(O.dd_permanent("glynn", a))
    print(f"c3a done {time.time() - t:.1f}s")
    b = W.c3b()
    if not skip_slow:
        t = time.time()
        k = O.prescale_factor(b)
        res["c3b_prescale"] = k
        res["c3b_ref_glynn_prescaled"] = enc(P.glynn_rectangular(b * k) / k ** b.shape[0])
        res["c3b_ref_glynn_raw"] = enc(P.glynn_rectangular(b))
        res["c3b_ref_ryser"] = enc(P.ryser_rectangular(b))
        print(f"c3b reference done {time.time() - t:.1f}s")
    t = time.time()
    res["c3b_dd_glynn"] = enc(O.dd_permanent("glynn", b))
    print(f"c3b dd done {time.time() - t:.1f}s")
    (OUT / "c3.json").write_text(json.dumps(res, indent=1) + "\n")


def gen_c4():
    res = {}
    for name, a in (("c4a", W.c4a()), ("c4b", W.c4b())):
        t = time.time()
        try:
            P.glynn(a)
            res[f"{name}_ref"] = "no-overflow"
        except OverflowError:
            res[f"{name}_ref"] = "OverflowError"
        try:
            P.ryser(a)
            res[f"{name}_ref_ryser"] = "no-overflow"
        except OverflowError:
            res[f"{name}_ref_ryser"] = "OverflowError"
        res[f"{name}_exact"] = str(O.exact_int128("glynn", a))
        print(f"{name}: {time.time() - t:.1f}s exact={res[name + '_exact']}")
    (OUT / "c4.json").write_text(json.dumps(res, indent=1) + "\n")


def gen_precision():
    """The reference's digits-lost table (src/oracles.py:160-236) at
    --max-n 16 --attempts 200 (SURVEY 8(f) item 2 baseline)."""
    from permanent.oracles import precision_csv, run_precision_suite

    t = time.time()
    recs = run_precision_suite(n_range=range(2, 17), seed=0, cauchy_attempts=200)
    (OUT / "precision_ref.csv").write_text(precision_csv(recs))
    print(f"precision_ref.csv: {len(recs)} rows, {time.time() - t:.1f}s")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-slow", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    OUT.mkdir(parents=True, exist_ok=True)
    O.build()
    steps = {"parity": gen_parity, "ref_cases": gen_ref_cases, "ref_int_walk": gen_ref_int_walk,
             "c1": gen_c1, "c2": gen_c2, "c3": lambda: gen_c3(args.skip_slow), "c4": gen_c4,
             "precision": gen_precision}
    for name, fn in steps.items():
        if args.only and name not in args.only.split(","):
            continue
        fn()


if __name__ == "__main__":
    main()
