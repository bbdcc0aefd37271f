"""Accuracy across the n-sweep (C5 law, seed 10 + n): FP64 Glynn (the timed
kernel) against the GPU double-double Ryser, both metrics of SURVEY 8(c)
-> profiles/r1_nsweep_accuracy.txt."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03421_b200 as P  # noqa: E402
from paper_2510_03421_b200 import engine as E, workloads as W  # noqa: E402
from paper_2510_03421_b200.algorithms import AlgorithmId  # noqa: E402
from paper_2510_03421_b200.core import as_matrix  # noqa: E402

for n in (20, 24, 28, 30, 32, 34, 36):
    a = W.c5(n)
    v, M = P.permanent_with_magsum(as_matrix(a), AlgorithmId.GLYNN)
    (rh, rl), _ = E.walk_dd("ryser", a)
    ref = rh + rl
    print(f"n={n}: glynn {v:.16e}  ryser_dd {ref:.16e}  rel {abs(v - ref) / abs(ref):.2e}  "
          f"scaled {abs(v - ref) / max(abs(v), abs(ref), M):.2e}  M/|per| {M / abs(ref):.2e}", flush=True)
