"""Quick GPU check: engine vs oracle on random matrices + a few timings."""
import ctypes as C, sys, time, math
import numpy as np
sys.path.insert(0, '.')
from paper_2510_03421_b200 import _lib as L
from oracle import oracle as O
lib = L.load()
rng = np.random.default_rng(1)
def call(name, a, mag=True):
    m, n = a.shape
    out = L.out_buf(2); mg = C.c_double()
    a = np.ascontiguousarray(a)
    st = getattr(lib, name)(m, n, L.ptr(a.view(np.float64) if np.iscomplexobj(a) else a), n, 0, out, C.byref(mg), None)
    L.check(st, name)
    v = complex(out[0], out[1]) if np.iscomplexobj(a) else out[0]
    return v, mg.value
worst = 0
for n in list(range(1, 15)) + [16, 18, 20]:
    for m in sorted(set([1, max(1, n // 2), n - 1 if n > 1 else 1, n])):
        for cplx in (False, True):
            a = rng.uniform(-1, 1, (m, n)) + (1j * rng.uniform(-1, 1, (m, n)) if cplx else 0)
            ref = O.dd_permanent("ryser", a, nthreads=8) if n <= 20 else None
            for alg in ("glynn", "ryser"):
                name = f"perm_{alg}_{'c128' if cplx else 'f64'}"
                v, mg = call(name, a)
                err = abs(v - ref) / max(abs(ref), mg, 1e-300)
                worst = max(worst, err)
                if err > 1e-12:
                    print("BAD", name, m, n, v, ref, mg, err)
print("worst scaled err", worst)
for n in (24, 28, 30, 32, 34, 36):
    a = rng.uniform(0, 1, (n, n)) / n
    call("perm_glynn_f64", a, mag=False)
    t = time.perf_counter(); v, _ = call("perm_glynn_f64", a, mag=False); dt = time.perf_counter() - t
    steps = 2 ** (n - 1)
    print(f"glynn f64 n={n}: {dt*1e3:.2f} ms  {steps/dt:.3e} steps/s  {steps*2*n/dt/1e12:.2f} Tops/s  val={v:.6e}")
for (m, n) in ((24, 24), (20, 28)):
    a = (rng.uniform(-1, 1, (m, n)) + 1j * rng.uniform(-1, 1, (m, n))) / math.sqrt(n)
    call("perm_glynn_c128", a)
    t = time.perf_counter(); v, mg = call("perm_glynn_c128", a, mag=False); dt = time.perf_counter() - t
    steps = 2 ** (n - 1)
    print(f"glynn c128 {m}x{n}: {dt*1e3:.2f} ms {steps/dt:.3e} steps/s {steps*(6*n-2)/dt/1e12:.2f} Tops/s val={v}")
a = rng.uniform(0, 1, (30, 30)) / 30
t = time.perf_counter(); v, _ = call("perm_ryser_f64", a); dt = time.perf_counter() - t
print(f"ryser f64 n=30 {dt*1e3:.2f} ms {2**30/dt:.3e} subsets/s")
