"""Workload for the ncu launch list of the small single walks (n-sweep end):
a few public-API calls per size; run under
    ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/ncu_small_walks.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03421_b200 as P  # noqa: E402
from paper_2510_03421_b200 import workloads as W  # noqa: E402

for n in (16, 20, 22, 24, 26, 28):
    a = W.c5(n)
    for _ in range(3):
        P.glynn(a)
    P.ryser(a)
