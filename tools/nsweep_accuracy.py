"""Accuracy across the n-sweep (C5 law, seed 10 + n): FP64 Glynn (the timed
kernel) against the GPU double-double Ryser, both metrics of SURVEY 8(c),
plus the C5 closed forms (J_36 = 36!, rank-one u v^T) and C3a / C3b against
the committed double-double values.  PERM_WALK_MAX_LOG2L selects the chunk
cap.  -> profiles/r2_nsweep_accuracy.txt"""
import json
import math
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2510_03421_b200 as P  # noqa: E402
from paper_2510_03421_b200 import engine as E, workloads as W  # noqa: E402
from paper_2510_03421_b200.algorithms import AlgorithmId  # noqa: E402
from paper_2510_03421_b200.core import as_matrix  # noqa: E402

print(f"# chunk cap 2^{os.environ.get('PERM_WALK_MAX_LOG2L', 'default')}", flush=True)
ns = [int(x) for x in sys.argv[1:]] or [20, 24, 28, 30, 32, 34, 36]
for n in ns:
    a = W.c5(n)
    t = time.perf_counter()
    v, M = P.permanent_with_magsum(as_matrix(a), AlgorithmId.GLYNN)
    (rh, rl), _ = E.walk_dd("ryser", a)
    ref = rh + rl
    print(f"n={n}: glynn {v:.16e}  ryser_dd {ref:.16e}  rel {abs(v - ref) / abs(ref):.2e}  "
          f"scaled {abs(v - ref) / max(abs(v), abs(ref), M):.2e}  M/|per| {M / abs(ref):.2e}", flush=True)
for name, (a, exact) in (("J_36", W.ones(36)), ("rank-one u v^T n=36", W.rank_one(36))):
    v, M = P.permanent_with_magsum(as_matrix(a), AlgorithmId.GLYNN)
    print(f"{name}: glynn {v:.16e}  exact {exact:.16e}  rel {abs(v - exact) / abs(exact):.2e}  "
          f"scaled {abs(v - exact) / max(abs(v), abs(exact), M):.2e}", flush=True)
c3 = json.loads((ROOT / "tests" / "golden" / "c3.json").read_text())
for name, a, key in (("C3a", W.c3a(), "c3a_dd_glynn"), ("C3b", W.c3b(), "c3b_dd_glynn")):
    d = c3[key]
    ref = complex(d["re"], d["im"])
    v, M = P.permanent_with_magsum(as_matrix(a), AlgorithmId.GLYNN)
    print(f"{name}: glynn {v:.16e}  dd {ref:.16e}  rel {abs(v - ref) / abs(ref):.2e}  "
          f"scaled {abs(v - ref) / max(abs(v), abs(ref), M):.2e}", flush=True)
