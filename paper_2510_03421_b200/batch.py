"""Batched permanents of many small matrices (north_star item 4).

The reference has no batch entry point -- ``as_matrix`` rejects anything but
2-D input (src/core.py:150-151) and callers loop in Python, one ~1-10 ms
``opt`` call per matrix.  These functions take a [B, m, n] array
(numpy on the host, or a torch CUDA tensor read in place) and evaluate all B
permanents with one kernel launch (C ABI perm_batch_*).  The batch dispatch
(``opt_batch``) uses two batch-only exact formulas that are cheaper per
matrix than any of the reference's algorithms: the set-partition (Moebius)
formula for m <= 6 and, for 8x8, the row-by-row subset recursion with its
middle level parked in tensor memory, both streamed through shared memory by
bulk copies (csrc/batch_bulk.cuh).

Integer batches return exact Python ints with the single-matrix semantics:
matrices whose magnitudes certify exact FP64 arithmetic run on the batch
kernels, the rest through the exact single-matrix path (``_int_batch``).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .algorithms import AlgorithmId

_ALG = {None: -1, "auto": -1, AlgorithmId.COMBINATORIC: 0, AlgorithmId.RYSER: 1, AlgorithmId.GLYNN: 2,
        "combinatoric": 0, "ryser": 1, "glynn": 2, "partition": 3, "laplace": 4}


def _run(a, alg):
    lib = _lib.load()
    code = _ALG[alg]
    try:
        import torch

        if isinstance(a, torch.Tensor) and a.is_cuda:
            if a.dim() != 3:
                raise TypeError("expected a [B, m, n] tensor")
            t = a
            if t.shape[1] > t.shape[2]:
                t = t.transpose(1, 2)
            if not t.is_complex():
                t = t.to(torch.float64)
            else:
                t = t.to(torch.complex128)
            t = t.contiguous()
            B, m, n = t.shape
            out = torch.empty(B, dtype=t.dtype, device=t.device)
            fn = lib.perm_batch_c128 if t.is_complex() else lib.perm_batch_f64
            st = fn(code, B, m, n, C.c_void_p(t.data_ptr()), C.c_void_p(out.data_ptr()), 1,
                    C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream))
            _lib.check(st, f"batch {B}x{m}x{n}")
            return out
    except ImportError:  # pragma: no cover
        pass
    arr = np.asarray(a)
    if arr.ndim != 3:
        raise TypeError(f"expected a [B, m, n] array, got ndim={arr.ndim}")
    if arr.shape[1] > arr.shape[2]:
        arr = np.swapaxes(arr, 1, 2)
    if arr.dtype.kind in "iub":
        return _int_batch(arr, code)
    cplx = np.iscomplexobj(arr)
    arr = np.ascontiguousarray(arr, dtype=np.complex128 if cplx else np.float64)
    B, m, n = arr.shape
    out = np.empty(B, dtype=arr.dtype)
    if B == 0:
        return out
    fn = lib.perm_batch_c128 if cplx else lib.perm_batch_f64
    st = fn(code, B, m, n, C.c_void_p(arr.ctypes.data), C.c_void_p(out.ctypes.data), 0, None)
    if st == _lib.BUDGET:
        from .algorithms import StepBudgetExceeded

        raise StepBudgetExceeded(_lib.last_error())
    _lib.check(st, f"batch {B}x{m}x{n}")
    return out


def _int_batch(arr, code):
    """Integer batches: exact Python ints with the single-matrix semantics.

    Matrices whose magnitudes certify that every intermediate of the batch
    formula is an integer below 2^52 run on the float batch kernels, where
    FP64 is then exact: the partition / 8x8 row-recursion formulas need
    m! * prod_i (row sum of |a|) < 2^52 (every partial sum is a signed sum of
    permanent monomials of |A|, weighted by at most m! in total), square
    Glynn needs 2^(n-1) * prod_j (column sum of |a|) < 2^52.  Under the same
    bounds none of the reference's checked int64 algorithms can overflow
    either, so the result equals the per-matrix call.  Every other matrix
    (and every explicit glynn / ryser / combinatoric request, which keeps its
    own overflow semantics) goes through the exact single-matrix path."""
    import math

    from . import combinatoric, glynn, opt, ryser

    per_matrix = {-1: opt, 0: combinatoric, 1: ryser, 2: glynn, 3: opt, 4: opt}[code]
    B, m, n = arr.shape
    out = np.empty(B, dtype=object)
    if B == 0:
        return out
    certified = np.zeros(B, dtype=bool)
    sel = int(_lib.load().perm_batch_select(m, n)) if code == -1 else code
    if code in (-1, 3, 4) and (sel in (3, 4) or (sel == 2 and m == n)):
        x = arr.astype(np.float64)
        ax = np.abs(x)
        with np.errstate(over="ignore", invalid="ignore"):
            if sel in (3, 4):
                bound = math.factorial(m) * np.prod(ax.sum(axis=2), axis=1)
            else:
                bound = 2.0 ** (n - 1) * np.prod(ax.sum(axis=1), axis=1)
        certified = np.isfinite(bound) & (bound < 2.0 ** 52)
        if certified.any():
            sub = np.ascontiguousarray(x[certified])
            vals = np.empty(sub.shape[0])
            fn = _lib.load().perm_batch_f64
            st = fn(sel, sub.shape[0], m, n, C.c_void_p(sub.ctypes.data), C.c_void_p(vals.ctypes.data), 0, None)
            _lib.check(st, f"batch {sub.shape[0]}x{m}x{n}")
            out[certified] = [int(v) for v in np.rint(vals)]
    for i in np.nonzero(~certified)[0]:
        out[i] = per_matrix(arr[i])
    return out


def opt_batch(a, params=None):
    """Permanents of a [B, m, n] batch with the batch dispatch
    (perm_batch_select: Laplace for 8x8 real, Glynn for other squares, the
    partition formula for m <= 4 < n and m = 5, 6 with n >= m + 2, Glynn on
    the ones-padded pre-scaled matrix for the other rectangles with n >= 9,
    subset-skipping Ryser otherwise).  Shapes: m <= n <= 30, and the
    partition formula up to n = 62.

    ``params`` (a TuningParams): the reference's selection rule
    (src/dispatch.py:84-95) picks one of combinatoric / Ryser / Glynn for the
    batch's shape instead, as ``opt(a, params=...)`` would per matrix."""
    if params is None:
        return _run(a, None)
    from .dispatch import select_algorithm

    shape = tuple(a.shape)
    if len(shape) != 3:
        raise TypeError(f"expected a [B, m, n] array, got ndim={len(shape)}")
    m, n = sorted(shape[1:])
    return _run(a, select_algorithm(m, n, params))


def partition_batch(a):
    """m <= 6 (complex m <= 5): sum over set partitions pi of the rows of
    mu(pi) prod_{blocks b} sum_j prod_{i in b} a_ij."""
    return _run(a, "partition")


def laplace_batch(a):
    """8x8 batch formula (the name is kept from round 1): the row-by-row
    subset recursion f_L(S) = sum_{j in S} a_{L-1,j} f_{L-1}(S \\ {j}),
    1016 FP64 ops per matrix (csrc/batch_bulk.cuh RowDp8Tm)."""
    return _run(a, "laplace")


def glynn_batch(a):
    return _run(a, "glynn")


def ryser_batch(a):
    return _run(a, "ryser")


def combinatoric_batch(a):
    return _run(a, "combinatoric")
