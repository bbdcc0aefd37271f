"""CPU oracle for the exact-permanent hot path -- TEST INFRASTRUCTURE ONLY.

Thin ctypes layer over ``oracle/libperm_oracle.so`` (built from
``perm_oracle.c`` by ``oracle/Makefile``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / reference arm
may import this module; the product package never does.

``permanent(alg, a)`` mirrors the reference wrappers in
``/root/reference/pkg/src/permanent/algorithms.py`` (``src/algorithms.py``
below) exactly -- same normalization arithmetic, same int64 overflow
semantics -- so float results are bit-identical to the reference's.

Parity pin: checked against the reference's 300 golden vectors
(``pkg/frontend/tests/fixtures/parity.json``, copied into
``tests/golden/parity.json``) and against fixtures made by running the
reference itself (``oracle/gen_golden.py``).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libperm_oracle.so"
_lib = None

COMBINATORIC, RYSER, GLYNN = "combinatoric", "ryser", "glynn"
INT64_MAX = 2**63 - 1
INT64_MIN = -(2**63)


def build() -> Path:
    """Compile the oracle library (idempotent)."""
    import subprocess

    src = _HERE / "perm_oracle.c"
    if not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = C.CDLL(str(_LIB_PATH))
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int64)
        for name in ("orc_comb_f64",):
            getattr(L, name).restype = C.c_double
            getattr(L, name).argtypes = [C.c_int, C.c_int, dp]
        L.orc_comb_c128.argtypes = [C.c_int, C.c_int, dp, dp]
        L.orc_comb_i64.argtypes = [C.c_int, C.c_int, ip, ip]
        L.orc_comb_i64.restype = C.c_int
        for name in ("orc_ryser_sq_f64", "orc_glynn_sq_f64"):
            getattr(L, name).restype = C.c_double
            getattr(L, name).argtypes = [C.c_int, dp]
        for name in ("orc_ryser_sq_c128", "orc_glynn_sq_c128"):
            getattr(L, name).argtypes = [C.c_int, dp, dp]
        for name in ("orc_ryser_sq_i64", "orc_glynn_sq_i64"):
            getattr(L, name).restype = C.c_int
            getattr(L, name).argtypes = [C.c_int, ip, ip]
        for name in ("orc_ryser_rect_f64", "orc_glynn_rect_f64"):
            getattr(L, name).restype = C.c_double
            getattr(L, name).argtypes = [C.c_int, C.c_int, dp]
        for name in ("orc_ryser_rect_c128", "orc_glynn_rect_c128"):
            getattr(L, name).argtypes = [C.c_int, C.c_int, dp, dp]
        for name in ("orc_ryser_rect_i64", "orc_glynn_rect_i64"):
            getattr(L, name).restype = C.c_int
            getattr(L, name).argtypes = [C.c_int, C.c_int, ip, ip]
        L.orc_walk_f64_range.restype = C.c_double
        L.orc_walk_f64_range.argtypes = [C.c_int, C.c_int, dp, dp, C.c_int, dp, C.c_uint64, C.c_uint64]
        L.orc_walk_mt.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_void_p]
        _lib = L
    return _lib


def _p(arr, ctype):
    return arr.ctypes.data_as(C.POINTER(ctype))


def _kind(a: np.ndarray) -> str:
    return {"i": "i64", "b": "i64", "u": "i64", "f": "f64", "c": "c128"}[a.dtype.kind]


def as_array(a) -> np.ndarray:
    """The reference's dtype mapping (src/core.py:29-47, 141-164)."""
    arr = np.asarray(a)
    k = arr.dtype.kind
    dt = {"b": np.int64, "i": np.int64, "u": np.int64, "f": np.float64, "c": np.complex128}[k]
    return np.ascontiguousarray(arr.astype(dt))


# ---------------------------------------------------------------------------
# raw kernels: the reference's get_kernel(name) contract (src/_kernels.py)
# ---------------------------------------------------------------------------

def kernel(name: str, a: np.ndarray):
    """Raw kernel value: float / complex, or (int, overflowed) for int64."""
    L = lib()
    a = np.ascontiguousarray(a)
    m, n = a.shape
    kind = _kind(a)
    base = {"comb_dfs": "comb", "ryser_sq": "ryser_sq", "ryser_rect": "ryser_rect",
            "glynn_sq": "glynn_sq", "glynn_rect": "glynn_rect"}[name]
    two_dim = base in ("comb", "ryser_rect", "glynn_rect")
    fn = getattr(L, f"orc_{base}_{kind}")
    args = (m, n) if two_dim else (n,)
    if kind == "f64":
        return float(fn(*args, _p(a, C.c_double)))
    if kind == "c128":
        out = np.zeros(2)
        fn(*args, _p(a.view(np.float64), C.c_double), _p(out, C.c_double))
        return np.complex128(complex(out[0], out[1]))
    out = np.zeros(1, np.int64)
    ovf = fn(*args, _p(a, C.c_int64), _p(out, C.c_int64))
    return int(out[0]), bool(ovf)


def _plain(value, kind):
    return float(value) if kind == "f64" else complex(value)


def permanent(alg: str, a, step_budget: int = 2_000_000_000, compiled=None):
    """(value, overflowed) exactly as ``run_algorithm`` (src/algorithms.py:187-201)
    returns it, for an m <= n matrix."""
    a = as_array(a)
    m, n = a.shape
    if m > n:
        raise ValueError("need m <= n")
    kind = _kind(a)
    if alg == COMBINATORIC:  # src/algorithms.py:71-90
        if math.perm(n, m) > step_budget:
            raise RuntimeError("step budget")
        r = kernel("comb_dfs", a)
        return r if kind == "i64" else (_plain(r, kind), False)
    if alg == RYSER:
        if m == n:  # src/algorithms.py:93-107
            r = kernel("ryser_sq", a)
        else:  # src/algorithms.py:118-137
            r = kernel("ryser_rect", a)
        return r if kind == "i64" else (_plain(r, kind), False)
    if alg == GLYNN:
        if m == n:  # src/algorithms.py:140-160
            if kind == "i64":
                acc, ovf = kernel("glynn_sq", a)
                if ovf:
                    return 0, True
                denom = 1 << (n - 1)
                if acc % denom:
                    return 0, True
                return acc // denom, False
            acc = kernel("glynn_sq", a)
            if kind == "f64":
                acc = np.float64(acc)
            return _plain(acc / (2.0 ** (n - 1)), kind), False
        # src/algorithms.py:163-184
        if kind == "i64":
            acc, ovf = kernel("glynn_rect", a)
            if ovf:
                return 0, True
            denom = (1 << (n - 1)) * math.factorial(n - m)
            if acc % denom:
                return 0, True
            return acc // denom, False
        acc = kernel("glynn_rect", a)
        if kind == "f64":
            acc = np.float64(acc)
        elif _compiled(1 << (n - 1), compiled):
            # numba hands back a Python complex, whose division by a float
            # is componentwise true division; the interpreted kernel's numpy
            # complex128 divides by multiplying with the reciprocal -- the two
            # modes differ in the last bit here (src/algorithms.py:182-183)
            acc = complex(acc)
        value = acc / (2.0 ** (n - 1)) / float(math.factorial(n - m))
        return _plain(value, kind), False
    raise ValueError(alg)


def _compiled(steps: int, compiled) -> bool:
    """src/algorithms.py:55-58: compiled kernels from 20 000 steps up."""
    return steps >= 20_000 if compiled is None else bool(compiled)


def brute_force(rows):
    """Exact permanent by permutation enumeration in Python arithmetic
    (the reference test suite's independent oracle, pkg/tests/conftest.py:13-26)."""
    import itertools

    rows = [list(r) for r in rows]
    m, n = len(rows), len(rows[0])
    if m > n:
        rows = [[rows[i][j] for i in range(m)] for j in range(n)]
        m, n = n, m
    total = 0
    for perm in itertools.permutations(range(n), m):
        p = 1
        for i in range(m):
            p *= rows[i][perm[i]]
        total += p
    return total


# ---------------------------------------------------------------------------
# Gray-range walks (perm_oracle.c section 2): sharded / higher precision
# ---------------------------------------------------------------------------

def walk_setup(alg: str, a: np.ndarray, scale: float = 1.0):
    """(P, B, v0, U, weights, norm) for the generic Gray walk of SURVEY App. A.

    Glynn works on the ones-padded n x n matrix with the real rows scaled by
    ``scale`` (a power of two; 1 reproduces the reference's Algorithm 4);
    Ryser-rectangular uses the all-subsets form with popcount weights.
    ``norm`` maps the walk sum to the permanent: per = sum * norm (exact
    rational as (num, den) in Python ints / floats)."""
    m, n = a.shape
    cplx = np.iscomplexobj(a)
    isint = a.dtype.kind in "iub"
    dt = np.int64 if isint else (np.complex128 if cplx else np.float64)
    if alg == GLYNN:
        full = np.ones((n, n), dt)
        full[:m] = a * scale if scale != 1.0 else a
        v0 = full.sum(axis=0)
        # U[t] = -2 * row (n-1-t), t = 0..n-2
        U = np.stack([-2 * full[n - 1 - t] for t in range(n - 1)]) if n > 1 else np.zeros((0, n), dt)
        return dict(P=n, B=n - 1, v0=np.ascontiguousarray(v0), U=np.ascontiguousarray(U),
                    weighted=False, w=None, m=m, n=n, alg=alg, scale=scale)
    if alg == RYSER:
        v0 = np.zeros(m, dt)
        U = np.ascontiguousarray(a.T.astype(dt))  # U[t] = column t
        if m == n:
            return dict(P=m, B=n, v0=v0, U=U, weighted=False, w=None, m=m, n=n, alg=alg, scale=1.0)
        w = [0] * (n + 1)
        for s in range(1, m + 1):
            w[s] = (-1) ** (m - s) * math.comb(n - s, m - s)
        return dict(P=m, B=n, v0=v0, U=U, weighted=True, w=w, m=m, n=n, alg=alg, scale=1.0)
    raise ValueError(alg)


def walk_f64_mt(setup, k0=0, k1=None, nthreads=None):
    """Sum of the walk terms over [k0, k1) in f64 (sequential per thread)."""
    L = lib()
    nthreads = nthreads or os.cpu_count() or 1
    k1 = (1 << setup["B"]) if k1 is None else k1
    v0 = np.ascontiguousarray(setup["v0"], np.float64)
    U = np.ascontiguousarray(setup["U"], np.float64)
    w = np.array(setup["w"] or [0.0], np.float64)
    out = np.zeros(2)
    L.orc_walk_mt(0, setup["P"], setup["B"], 0, int(setup["weighted"]), v0.ctypes.data, U.ctypes.data,
                  w.ctypes.data, k0, k1, nthreads, out.ctypes.data)
    return float(out[0]) + float(out[1])


def walk_dd_mt(setup, k0=0, k1=None, nthreads=None, mag=False):
    """Double-double walk sum over [k0, k1): returns (hi, lo) pairs
    ((re_hi, re_lo), (im_hi, im_lo)); with ``mag`` also the raw magnitude
    sum sum_k |w_k term_k| (dd-accumulated, rounded)."""
    L = lib()
    nthreads = nthreads or os.cpu_count() or 1
    k1 = (1 << setup["B"]) if k1 is None else k1
    cplx = np.iscomplexobj(setup["v0"]) or np.iscomplexobj(setup["U"])
    dt = np.complex128 if cplx else np.float64
    v0 = np.ascontiguousarray(setup["v0"], dt)
    U = np.ascontiguousarray(setup["U"], dt)
    w = np.array(setup["w"] or [0.0], np.float64)
    out = np.zeros(6)
    L.orc_walk_mt(1, setup["P"], setup["B"], int(cplx), int(setup["weighted"]), v0.ctypes.data,
                  U.ctypes.data, w.ctypes.data, k0, k1, nthreads, out.ctypes.data)
    if mag:
        return (out[0], out[1]), (out[2], out[3]), out[4] + out[5]
    return (out[0], out[1]), (out[2], out[3])


def walk_i128_mt(setup, k0=0, k1=None, nthreads=None) -> int:
    """Exact walk sum mod 2^128 over [k0, k1), as a signed Python int."""
    L = lib()
    nthreads = nthreads or os.cpu_count() or 1
    k1 = (1 << setup["B"]) if k1 is None else k1
    v0 = np.ascontiguousarray(setup["v0"], np.int64)
    U = np.ascontiguousarray(setup["U"], np.int64)
    w = np.array(setup["w"] or [0], np.int64)
    out = np.zeros(2, np.uint64)
    L.orc_walk_mt(2, setup["P"], setup["B"], 0, int(setup["weighted"]), v0.ctypes.data, U.ctypes.data,
                  w.ctypes.data, k0, k1, nthreads, out.ctypes.data)
    v = int(out[0]) | (int(out[1]) << 64)
    return v - (1 << 128) if v >= (1 << 127) else v


def exact_int128(alg: str, a, nthreads=None) -> int:
    """Exact permanent of an integer matrix via the wrapping-int128 walk
    (valid when the true walk sum lies in (-2^127, 2^127))."""
    a = as_array(a)
    m, n = a.shape
    s = walk_setup(alg, a)
    total = walk_i128_mt(s, nthreads=nthreads)
    # The int128 walk wraps silently.  Guard with the double-double value of
    # the same walk: refuse when the walk sum (the permanent times Glynn's
    # 2^(n-1) (n-m)!) is not safely inside int128.
    denom = (1 << (n - 1)) * math.factorial(n - m) if alg == GLYNN else 1
    est = abs(dd_permanent(alg, np.asarray(a, dtype=np.float64), nthreads=nthreads)) * float(denom)
    if not est < 2.0 ** 126:
        raise OverflowError(f"oracle: the {alg} int128 walk sum (~{est:.3e}) does not fit; use the other algorithm")
    if alg == GLYNN:
        assert total % denom == 0
        return total // denom
    if m == n:
        return -total if n & 1 else total
    return total


def dd_permanent(alg: str, a, scale=None, nthreads=None):
    """Double-double permanent (the 'higher-precision restatement' of
    SURVEY 8(c)); returns a Python float or complex (rounded from dd)."""
    a = as_array(a).astype(np.complex128 if np.iscomplexobj(a) else np.float64)
    m, n = a.shape
    if scale is None:
        scale = prescale_factor(a) if (alg == GLYNN and m < n) else 1.0
    s = walk_setup(alg, a, scale=scale)
    (rh, rl), (ih, il) = walk_dd_mt(s, nthreads=nthreads)
    if alg == GLYNN:
        norm = 2.0 ** (n - 1) * float(math.factorial(n - m)) * scale ** m
        re, im = (rh + rl) / norm, (ih + il) / norm
    else:
        sign = -1.0 if (m == n and n & 1) else 1.0
        re, im = sign * (rh + rl), sign * (ih + il)
    return complex(re, im) if np.iscomplexobj(a) else re


def prescale_factor(a: np.ndarray) -> float:
    """Power of two k ~ 1/RMS of the nonzero |a_ij|: the
    rectangular-Glynn conditioning fix.  Same rule as the engine."""
    mag2 = np.abs(a) ** 2
    nz = mag2[mag2 != 0]
    if nz.size == 0:
        return 1.0
    rms = float(np.sqrt(np.mean(nz)))
    if not np.isfinite(rms) or rms == 0.0:
        return 1.0
    return float(2.0 ** round(-math.log2(rms)))


def ryser_magnitude_sum(a: np.ndarray, nthreads=None) -> float:
    """Ryser's magnitude sum sum_S |w_S prod_i rowsum_i(S)| (the all-subsets
    form, double-double walk): the scale for Ryser of a permanent that is
    exactly 0, where Glynn's M can vanish while Ryser leaves O(eps M_R)."""
    a = as_array(a)
    a = a.astype(np.complex128 if np.iscomplexobj(a) else np.float64)
    _, _, mg = walk_dd_mt(walk_setup(RYSER, a), nthreads=nthreads, mag=True)
    return float(mg)


def glynn_magnitude_sum(a: np.ndarray, scale=None, nthreads=None) -> float:
    """M = norm * sum_k |prod_j colsum_j(k)|: by brute
    walk in numpy for n <= 14, else the C double-double walk (threads)."""
    a = as_array(a)
    m, n = a.shape
    if scale is None:
        scale = prescale_factor(a) if m < n else 1.0
    if n > 14:
        s = walk_setup(GLYNN, a.astype(np.complex128 if np.iscomplexobj(a) else np.float64), scale=scale)
        _, _, mg = walk_dd_mt(s, nthreads=nthreads, mag=True)
        return float(mg / (2.0 ** (n - 1) * math.factorial(n - m) * scale ** m))
    full = np.ones((n, n), np.complex128 if np.iscomplexobj(a) else np.float64)
    full[:m] = a * scale
    K = 1 << (n - 1)
    ks = np.arange(K, dtype=np.int64)
    g = ks ^ (ks >> 1)
    delta = np.ones((K, n))
    for t in range(n - 1):
        delta[:, n - 1 - t] = np.where((g >> t) & 1, -1.0, 1.0)
    colsums = delta @ full
    mag = np.abs(np.prod(colsums, axis=1)).sum()
    return float(mag / (2.0 ** (n - 1) * math.factorial(n - m) * scale ** m))
