"""Per-call latency breakdown for small single permanents."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03421_b200 as P
from paper_2510_03421_b200 import _lib
from paper_2510_03421_b200.algorithms import permanent_glynn_square
from paper_2510_03421_b200.core import as_matrix

lib = _lib.load()
a = np.random.default_rng(0).uniform(-1, 1, (12, 12))
out = _lib.out_buf(2)


def t(fn, n=2000):
    for _ in range(50):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


ptr = C.c_void_p(a.ctypes.data)
print("raw ctypes perm_glynn_f64 12x12: %.1f us" % t(lambda: lib.perm_glynn_f64(12, 12, ptr, 12, 0, out, None, None)))
m = as_matrix(a)
print("permanent_glynn_square(Matrix): %.1f us" % t(lambda: permanent_glynn_square(m)))
print("P.glynn(ndarray): %.1f us" % t(lambda: P.glynn(a)))
print("as_matrix: %.1f us" % t(lambda: as_matrix(a)))
b = np.random.default_rng(0).uniform(-1, 1, (6, 6))
pb = C.c_void_p(b.ctypes.data)
print("raw ctypes perm_glynn_f64 6x6 (batch-of-one path): %.1f us" % t(lambda: lib.perm_glynn_f64(6, 6, pb, 6, 0, out, None, None)))
c = np.random.default_rng(0).uniform(-1, 1, (20, 20))
pc = C.c_void_p(c.ctypes.data)
print("raw ctypes perm_glynn_f64 20x20: %.1f us" % t(lambda: lib.perm_glynn_f64(20, 20, pc, 20, 0, out, None, None), 500))
