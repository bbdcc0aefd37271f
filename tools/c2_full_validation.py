"""All 1e6 matrices of C2a / C2b: the batch-only formulas (row recursion 8x8,
set partitions 4x10) against the classic per-matrix kernels (Glynn /
memoized combinatoric), with the error scaled by per(|A|) (the permanent's
own magnitude sum, computed with the same kernels on |A|, where nothing
cancels) -> profiles/r1_c2_full_validation.txt."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03421_b200 as P  # noqa: E402
from paper_2510_03421_b200 import workloads as W  # noqa: E402

for name, A, fast, classic in (("C2a 1e6 x 8x8", W.c2a(), P.laplace_batch, P.glynn_batch),
                              ("C2b 1e6 x 4x10", W.c2b(), P.partition_batch, P.combinatoric_batch)):
    x = fast(A)
    r = classic(A)
    mag = fast(np.abs(A))
    scale = np.maximum(np.maximum(np.abs(x), np.abs(r)), mag)
    err = np.abs(x - r) / scale
    rel = np.abs(x - r) / np.maximum(np.maximum(np.abs(x), np.abs(r)), 1e-300)
    print(f"{name}: max |fast - classic| / per(|A|) = {err.max():.3e} (mean {err.mean():.2e}); "
          f"cells over 1e-10: {(err > 1e-10).sum()}; plain relative max {rel.max():.2e}, "
          f"over 1e-10 relative: {(rel > 1e-10).sum()} (near-zero permanents)")
