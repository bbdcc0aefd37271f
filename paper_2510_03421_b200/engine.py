"""Typed calls into the C ABI (include/permanent_b200.h).

This module is the replacement of the reference's kernel registry
``_kernels.get_kernel`` (/root/reference/pkg/src/permanent/_kernels.py:718-728):
the reference returns a raw enumeration kernel and normalizes in
``algorithms.py``; here each call returns the normalized permanent computed
on the GPU.  Arrays are host numpy arrays (staged by the engine) or torch
CUDA tensors (read in place).
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib

ALG_CODE = {"combinatoric": _lib.ALG_COMBINATORIC, "ryser": _lib.ALG_RYSER, "glynn": _lib.ALG_GLYNN}


def _stage(a):
    """(pointer, lda, dev_ptr, keepalive, stream) for a 2-D array or tensor."""
    if isinstance(a, np.ndarray) and a.flags.c_contiguous:  # the common case, no torch lookup
        return C.c_void_p(a.ctypes.data), a.shape[1], 0, a, None
    try:
        import torch

        if isinstance(a, torch.Tensor) and a.is_cuda:
            t = a.contiguous()
            if t.dtype == torch.complex128:
                lda = t.shape[1]
            else:
                lda = t.shape[1]
            return C.c_void_p(t.data_ptr()), lda, 1, t, C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)
    except ImportError:  # pragma: no cover
        pass
    arr = np.ascontiguousarray(a)
    return C.c_void_p(arr.ctypes.data), arr.shape[1], 0, arr, None


def _kind(a) -> str:
    """numpy dtype kind character of an array or tensor ('i', 'f', 'c')."""
    if isinstance(a, np.ndarray):
        return a.dtype.kind
    if a.is_complex():
        return "c"
    return "f" if a.is_floating_point() else "i"


_WALK_FN = {}  # (alg, complex) -> bound C entry point


def walk(alg: str, a, magsum: bool = False):
    """Glynn / Ryser permanent of a float64 or complex128 m x n (m <= n)
    matrix; returns (value, M) with M the magnitude sum (or None)."""
    cplx = _kind(a) == "c"
    m, n = a.shape
    ptr, lda, dev, keep, stream = _stage(a)
    out = _lib.out_buf(2)
    fn = _WALK_FN.get((alg, cplx))
    if fn is None:
        fn = _WALK_FN[(alg, cplx)] = getattr(_lib.load(), f"perm_{alg}_{'c128' if cplx else 'f64'}")
    if magsum:
        mg = C.c_double(0.0)
        st = fn(m, n, ptr, lda, dev, out, C.byref(mg), stream)
    else:
        st = fn(m, n, ptr, lda, dev, out, None, stream)
    _lib.check(st, f"{alg} {m}x{n}")
    val = complex(out[0], out[1]) if cplx else float(out[0])
    return val, (mg.value if magsum else None)


_FAST_DTYPES = {np.dtype(np.float64): False, np.dtype(np.complex128): True}
_TLS = threading.local()  # per-thread result buffer (ctypes releases the GIL during the call)


def walk_host_fast(alg: str, a):
    """The public glynn / ryser call on a host float64 / complex128 2-D
    C-contiguous array with m <= n <= 62, without the Matrix wrapper: the
    per-call Python cost drops from ~10 to ~3 us (the result is the same
    engine call as ``walk``).  Returns None when the fast path does not
    apply."""
    cplx = _FAST_DTYPES.get(a.dtype)
    if cplx is None or a.ndim != 2 or not a.flags.c_contiguous:
        return None
    m, n = a.shape
    if m < 1 or m > n or n > 62:
        return None
    fn = _WALK_FN.get((alg, cplx))
    if fn is None:
        fn = _WALK_FN[(alg, cplx)] = getattr(_lib.load(), f"perm_{alg}_{'c128' if cplx else 'f64'}")
    out = getattr(_TLS, "out", None)
    if out is None:
        out = _TLS.out = _lib.out_buf(2)
    st = fn(m, n, a.ctypes.data, n, 0, out, None, None)
    if st:
        _lib.check(st, f"{alg} {m}x{n}")
    return complex(out[0], out[1]) if cplx else out[0]


def comb(a, step_budget: int, width: int = 64):
    """Combinatoric permanent (float64 / complex128 / integer).
    Returns (value, overflowed, status).  Integers: width=64 is the
    reference's checked int64 (overflowed as it reports it); width=128 the
    exact int128 DFS, overflowed = "does not fit int64", OverflowError when
    the int128 bound fails.  BUDGET is mapped by the caller."""
    lib = _lib.load()
    m, n = a.shape
    kind = _kind(a)
    ptr, lda, dev, keep, stream = _stage(a)
    budget = C.c_uint64(min(int(step_budget), (1 << 64) - 1) if step_budget >= 0 else 0)
    if kind in ("i",):
        out = (C.c_int64 * 2)()
        fits = C.c_int(1)
        st = lib.perm_comb_i64(m, n, ptr, lda, dev, width, budget, out, C.byref(fits), stream)
        if st == _lib.OVERFLOW:
            if width == 64:
                return 0, True, st
            raise OverflowError(f"exact int128 combinatoric {m}x{n}: {_lib.last_error()}")
        if st == _lib.BUDGET:
            return None, False, st
        _lib.check(st, f"combinatoric {m}x{n}")
        v = (int(out[1]) << 64) | (int(out[0]) & ((1 << 64) - 1))
        return v, (width == 128 and not fits.value), st
    cplx = kind == "c"
    out = _lib.out_buf(2)
    fn = lib.perm_comb_c128 if cplx else lib.perm_comb_f64
    st = fn(m, n, ptr, lda, dev, budget, out, stream)
    if st == _lib.BUDGET:
        return None, False, st
    _lib.check(st, f"combinatoric {m}x{n}")
    return (complex(out[0], out[1]) if cplx else float(out[0])), False, st


def exact_int(alg: str, a: np.ndarray, width: int = 64):
    """Integer permanent.  width=64: (value, overflowed) with the reference's
    checked-int64 semantics; width=128: (exact int, not fits_int64), raising
    OverflowError when the int128 fit certificate fails."""
    lib = _lib.load()
    m, n = a.shape
    ptr, lda, dev, keep, stream = _stage(a)
    out = (C.c_int64 * 2)()
    fits = C.c_int(0)
    fn = lib.perm_glynn_i64 if alg == "glynn" else lib.perm_ryser_i64
    st = fn(m, n, ptr, lda, dev, width, out, C.byref(fits), stream)
    if st == _lib.OVERFLOW:
        if width == 64:
            return 0, True
        raise OverflowError(f"exact int128 {alg} {m}x{n}: {_lib.last_error()}")
    _lib.check(st, f"{alg} int{width} {m}x{n}")
    v = (int(out[1]) << 64) | (int(out[0]) & ((1 << 64) - 1))
    return v, (not fits.value)


def walk_dd(alg: str, a):
    """Double-double Glynn / Ryser on the GPU (validation): returns
    ((re_hi, re_lo), (im_hi, im_lo)) of the normalized permanent."""
    lib = _lib.load()
    if not isinstance(a, np.ndarray):  # validation walk: host copy of a device matrix
        a = a.cpu().numpy()
    cplx = np.iscomplexobj(a)
    a = np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)
    m, n = a.shape
    out = _lib.out_buf(4)
    st = lib.perm_permanent_dd(ALG_CODE[alg], int(cplx), m, n, C.c_void_p(a.ctypes.data), n, 0, out, None)
    _lib.check(st, f"dd {alg} {m}x{n}")
    return (out[0], out[1]), (out[2], out[3])


def walk_steps(alg: str, m: int, n: int) -> int:
    return int(_lib.load().perm_walk_steps(ALG_CODE[alg], m, n))


def sm_count() -> int:
    return int(_lib.load().perm_device_sm_count())


def ryser_rect(a):
    """The reference's ryser_rect kernel (lexicographic combination order,
    any m <= n incl. square, n <= 256): (value, overflowed); integers with
    the reference's checked int64 flag (src/_kernels.py:226-365)."""
    lib = _lib.load()
    m, n = a.shape
    kind = _kind(a)
    ptr, lda, dev, keep, stream = _stage(a)
    if kind == "i":
        out = (C.c_int64 * 2)()
        st = lib.perm_ryser_rect_i64(m, n, ptr, lda, dev, out, stream)
        if st == _lib.OVERFLOW:
            return 0, True
        _lib.check(st, f"ryser_rect {m}x{n}")
        return int(out[0]), False
    out = _lib.out_buf(2)
    fn = lib.perm_ryser_rect_c128 if kind == "c" else lib.perm_ryser_rect_f64
    _lib.check(fn(m, n, ptr, lda, dev, out, stream), f"ryser_rect {m}x{n}")
    return (complex(out[0], out[1]) if kind == "c" else float(out[0])), False
