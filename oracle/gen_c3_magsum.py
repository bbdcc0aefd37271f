"""Adds the oracle's magnitude sums M (SURVEY 8(c) metric (ii) scale) of the
C3a / C3b matrices to tests/golden/c3.json, so the GPU parity tests take M
from the oracle instead of the engine under test.  The C
double-double walk (oracle/perm_oracle.c orc_walk_dd_range) over all 2^23 /
2^27 Gray steps, threads = all host cores.  Test infrastructure only."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402
from paper_2510_03421_b200 import workloads as W  # noqa: E402

path = ROOT / "tests" / "golden" / "c3.json"
c3 = json.loads(path.read_text())
for key, a in (("c3a_glynn_magsum", W.c3a()), ("c3b_glynn_magsum", W.c3b())):
    t = time.perf_counter()
    c3[key] = O.glynn_magnitude_sum(a)
    print(key, c3[key], f"{time.perf_counter() - t:.1f} s", flush=True)
path.write_text(json.dumps(c3, indent=1) + "\n")
