"""Device-resident C2a / C2b batches (for ncu): 2 launches each."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2510_03421_b200 as P
from paper_2510_03421_b200 import workloads as W
for A in (W.c2a(), W.c2b()):
    dA = torch.tensor(A, device="cuda")
    for _ in range(2):
        P.opt_batch(dA)
    torch.cuda.synchronize()
print("ok")
