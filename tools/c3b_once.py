import sys
sys.path.insert(0, '.')
import paper_2510_03421_b200 as P
from paper_2510_03421_b200 import workloads as W
a = W.c3b()
for _ in range(3):
    P.glynn(a)
