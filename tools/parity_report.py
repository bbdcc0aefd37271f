"""Both parity metrics of SURVEY 8(c) for every BASELINE config, on the GPU
engine: (i) rel = |x - ref| / max(|x|, |ref|) and (ii) scaled = |x - ref| /
max(|x|, |ref|, M), M from the ORACLE (numpy / C double-double walk, or the
committed fixture it produced).  -> profiles/r2_parity_metrics.txt"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2510_03421_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2510_03421_b200 import engine as E, workloads as W  # noqa: E402

G = ROOT / "tests" / "golden"


def metrics(x, ref, M):
    x, ref, M = np.asarray(x), np.asarray(ref), np.asarray(M)
    d = np.abs(x - ref)
    rel = d / np.maximum(np.maximum(np.abs(x), np.abs(ref)), 1e-300)
    sc = d / np.maximum(np.maximum(np.abs(x), np.abs(ref)), np.maximum(M, 1e-300))
    return rel, sc


def line(name, rel, sc, note=""):
    rel, sc = np.atleast_1d(rel), np.atleast_1d(sc)
    print(f"{name:34s} n={rel.size:6d}  (i) max {rel.max():.2e}  >1e-10: {(rel > 1e-10).sum():4d}   "
          f"(ii) max {sc.max():.2e}  >1e-10: {(sc > 1e-10).sum():4d}  {note}", flush=True)


c1 = np.load(G / "c1.npz")
M1 = np.array([O.glynn_magnitude_sum(a) for a in c1["a"]])
for alg, fn in (("glynn", P.glynn), ("ryser", P.ryser), ("opt", P.opt)):
    got = np.array([fn(a) for a in c1["a"]])
    line(f"C1 {alg} vs reference {alg}", *metrics(got, c1[alg], M1))
got = P.glynn_batch(c1["a"])
line("C1 glynn_batch vs reference glynn", *metrics(got, c1["glynn"], M1))

c2 = np.load(G / "c2_sub.npz")
for A, key, name in ((W.c2a(), "8", "C2a"), (W.c2b(), "4", "C2b")):
    out = P.opt_batch(A)[:512]
    for ref in ("opt", "c", "r", "g"):
        line(f"{name} opt_batch[:512] vs ref {ref}", *metrics(out, c2[ref + key], c2["m" + key]),
             "(M: oracle, fixture)")

c3 = json.loads((G / "c3.json").read_text())
for name, a, dd, mk in (("C3a", W.c3a(), "c3a_dd_glynn", "c3a_glynn_magsum"),
                        ("C3b", W.c3b(), "c3b_dd_glynn", "c3b_glynn_magsum")):
    ref = complex(c3[dd]["re"], c3[dd]["im"])
    for fn in (P.glynn, P.ryser, P.opt):
        line(f"{name} {fn.__name__} vs dd oracle", *metrics(fn(a), ref, c3[mk]))

c4 = json.loads((G / "c4.json").read_text())
for name, a in (("c4a", W.c4a()), ("c4b", W.c4b())):
    ex = int(c4[f"{name}_exact"])
    ok = P.glynn(a, exact="int128") == ex and P.ryser(a, exact="int128") == ex
    print(f"{name.upper()} exact int128 glynn == ryser == fixture: {ok}")

c5 = json.loads((G / "c5_dd.json").read_text())
for n in (20, 24, 28, 30, 32, 34, 36):
    a = W.c5(n)
    ref = c5["ryser_dd"][str(n)]
    M = O.glynn_magnitude_sum(a) if n <= 24 else c5["glynn_magsum"].get(str(n), abs(ref))
    line(f"C5 n={n} glynn vs GPU dd Ryser", *metrics(P.glynn(a), ref, M),
         "(M: oracle)" if n <= 24 else "(M: fixture or |ref|; (i) is the bar)")
for name, (a, ex) in (("J_36", W.ones(36)), ("u v^T n=36", W.rank_one(36))):
    line(f"C5 {name} glynn vs closed form", *metrics(P.glynn(a), ex, abs(ex)))
