"""One C4a exact int128 Glynn call (for ncu): gpurun -- python tools/c4a_once.py"""
import sys
sys.path.insert(0, '.')
import paper_2510_03421_b200 as P
from paper_2510_03421_b200 import workloads as W
x = W.c4a()
for _ in range(2):
    print(P.glynn(x, exact="int128"))
