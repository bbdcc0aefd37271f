"""C3a (complex 24x24 Glynn) and C4a (0/1 32x32 exact int128 Glynn), 2 calls each (for ncu)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03421_b200 as P
from paper_2510_03421_b200 import workloads as W
a, b = W.c3a(), W.c4a()
for _ in range(2):
    P.glynn(a)
    P.glynn(b, exact="int128")
print("ok")
