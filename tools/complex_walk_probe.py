"""Complex128 Glynn walks n = 24..33: device time per permanent
(perm_walk_repeat_ms) and the fraction of the FP64 pipe (6n - 2 ops per
step, DADD/DMUL probe peak) -- the spill onset of the complex walk (P >= 30).

    python tools/complex_walk_probe.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_03421_b200 import _lib  # noqa: E402

lib = _lib.load()
peak = _lib.out_buf(1)
_lib.check(lib.perm_fp64_pipe_probe(1, 0.5, peak), "probe")
rng = np.random.default_rng(0)
for n in range(24, 34):
    a = np.ascontiguousarray((rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))) / np.sqrt(n))
    ms = _lib.out_buf(1)
    reps = 20 if n <= 28 else 3
    _lib.check(lib.perm_walk_repeat_ms(_lib.ALG_GLYNN, 1, n, n, _lib.C.c_void_p(a.ctypes.data), n, reps, ms), "rep")
    steps = 2 ** (n - 1)
    print(f"c128 n={n}: {ms[0]:10.3f} ms  {steps / (ms[0] * 1e-3):.3e} steps/s  "
          f"pipe {steps * (6 * n - 2) / (ms[0] * 1e-3) / peak[0]:.1%}", flush=True)
