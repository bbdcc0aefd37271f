"""Accuracy report for the large configs (C3, C4, C5) -> stdout / profiles.

Prints, per config, the engine value, the cross-checks and both error
metrics ((i) relative, (ii) scaled by the magnitude sum M).
"""
from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2510_03421_b200 as P  # noqa: E402
from paper_2510_03421_b200 import engine as E, workloads as W  # noqa: E402
from paper_2510_03421_b200.algorithms import AlgorithmId  # noqa: E402
from paper_2510_03421_b200.core import as_matrix  # noqa: E402


def dd(a, alg):
    (rh, rl), (ih, il) = E.walk_dd(alg, a)
    return complex(rh + rl, ih + il) if np.iscomplexobj(a) else rh + rl


def errs(x, ref, M):
    rel = abs(x - ref) / max(abs(x), abs(ref), 1e-300)
    sc = abs(x - ref) / max(abs(x), abs(ref), M, 1e-300)
    return rel, sc


def main():
    out = {}
    golden = ROOT / "tests" / "golden"
    c3 = json.loads((golden / "c3.json").read_text())
    c4 = json.loads((golden / "c4.json").read_text())

    a = W.c5(36)
    v, M = P.permanent_with_magsum(as_matrix(a), AlgorithmId.GLYNN)
    r, g = dd(a, "ryser"), dd(a, "glynn")
    out["C5 n=36 Glynn f64 vs Ryser dd (GPU)"] = (v, r, M) + errs(v, r, M)
    out["C5 n=36 Glynn dd vs Ryser dd (GPU)"] = (g, r, M) + errs(g, r, M)
    j, exact = W.ones(36)
    v, M = P.permanent_with_magsum(as_matrix(j), AlgorithmId.GLYNN)
    out["J_36 Glynn f64 vs 36!"] = (v, exact, M) + errs(v, exact, M)
    u, exact = W.rank_one(36)
    v, M = P.permanent_with_magsum(as_matrix(u), AlgorithmId.GLYNN)
    out["rank-one u v^T n=36 Glynn f64 vs 36! prod(u) prod(v)"] = (v, exact, M) + errs(v, exact, M)

    def cdec(d):
        return complex(d["re"], d["im"])

    a = W.c3a()
    v, M = P.permanent_with_magsum(as_matrix(a), AlgorithmId.GLYNN)
    for name, ref in (("dd oracle (CPU)", cdec(c3["c3a_dd_glynn"])), ("reference glynn", cdec(c3["c3a_ref_glynn"])),
                      ("reference ryser", cdec(c3["c3a_ref_ryser"]))):
        out[f"C3a Glynn c128 vs {name}"] = (v, ref, M) + errs(v, ref, M)
    b = W.c3b()
    v, M = P.permanent_with_magsum(as_matrix(b), AlgorithmId.GLYNN)
    refs = [("dd oracle (CPU)", cdec(c3["c3b_dd_glynn"]))]
    if "c3b_ref_glynn_prescaled" in c3:
        refs += [("reference glynn on pre-scaled matrix", cdec(c3["c3b_ref_glynn_prescaled"])),
                 ("reference ryser-rect", cdec(c3["c3b_ref_ryser"])),
                 ("reference glynn-rect (unscaled, SURVEY 0.5c)", cdec(c3["c3b_ref_glynn_raw"]))]
    for name, ref in refs:
        out[f"C3b Glynn c128 vs {name}"] = (v, ref, M) + errs(v, ref, M)

    for name, a in (("C4a", W.c4a()), ("C4b", W.c4b())):
        exact = int(c4[f"{name.lower()}_exact"])
        g = P.glynn(a, exact="int128")
        rr = P.ryser(a, exact="int128")
        out[f"{name} int128 Glynn / Ryser vs oracle exact"] = (str(g), str(rr), str(exact), g == exact == rr)

    lines = []
    for k, val in out.items():
        if len(val) == 5:
            x, ref, M, rel, sc = val
            lines.append(f"{k}:\n    value {x}\n    ref   {ref}\n    M {M:.6g}  rel {rel:.3e}  scaled {sc:.3e}")
        else:
            lines.append(f"{k}: glynn={val[0]} ryser={val[1]} exact={val[2]} equal={val[3]}")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
