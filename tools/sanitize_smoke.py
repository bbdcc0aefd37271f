"""Small invocations of every kernel family (bulk pipelines with ragged
last tiles, classic batch kernels, batched medium walks, zero-copy single
calls, device-wide walks, exact and double-double paths), e.g. for
compute-sanitizer where it is available (it is closed on this round's GPU
pool; the parity tests compare every family with the oracle instead):

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03421_b200 as P  # noqa: E402
from paper_2510_03421_b200 import sharded as S  # noqa: E402

rng = np.random.default_rng(5)
# bulk pipelines, ragged last tiles
P.partition_batch(rng.standard_normal((333, 4, 10)))
P.partition_batch(rng.standard_normal((77, 6, 8)))
P.partition_batch(rng.standard_normal((45, 3, 5)) + 1j * rng.standard_normal((45, 3, 5)))
P.laplace_batch(rng.standard_normal((97, 8, 8)))
# classic batch kernels and the warp-per-matrix Glynn
P.glynn_batch(rng.standard_normal((50, 6, 6)))
P.glynn_batch(rng.standard_normal((20, 12, 12)))
P.ryser_batch(rng.standard_normal((40, 5, 9)))
P.combinatoric_batch(rng.standard_normal((40, 3, 7)))
# medium batched walks (segments per matrix)
P.glynn_batch(rng.uniform(-1, 1, (3, 18, 18)) / 18)
# zero-copy single calls
P.glynn(rng.standard_normal((6, 6)))
P.glynn(rng.standard_normal((3, 7)))
P.glynn(rng.standard_normal((11, 11)))
P.combinatoric(rng.standard_normal((4, 9)))
# device-wide walks (U[0] in registers for real P >= 17), complex, weighted, dd, exact
P.glynn(rng.uniform(-1, 1, (20, 20)) / 20)
P.ryser(rng.uniform(-1, 1, (18, 18)) / 18)
P.glynn(rng.uniform(-1, 1, (16, 16)) + 1j * rng.uniform(-1, 1, (16, 16)))
P.ryser(rng.uniform(-1, 1, (12, 16)) / 16)
P.glynn((rng.random((20, 20)) < 0.5).astype(np.int64), exact="int128")
P.ryser(rng.integers(-2, 3, (14, 14)))
P.combinatoric(rng.standard_normal((9, 9)))
S.gpu_partial("glynn", rng.uniform(-1, 1, (24, 24)) / 24, 1 << 20, 1 << 21, mag=True)
print("sanitize smoke ok")
