"""Seeded fuzz with harsh value laws (heavy columns and rows, wide dynamic
range, exact zeros, integer-valued floats, near-singular structure) through
every single-matrix entry point, float and integer, against the CPU oracle.
Needs a B200.

Float: metric (ii) <= 1e-10 with M = the larger of the oracle's Glynn and
Ryser magnitude sums.  Integer: bit-exact values and the
reference's OverflowError on exactly the same inputs.
PERM_FUZZ_HARSH cases (default 120)."""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

import paper_2510_03421_b200 as P
from conftest import scaled_err
from oracle import oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-10


def harsh(rng, m, n, law):
    a = rng.uniform(-1, 1, (m, n))
    if law == 0:  # one heavy column
        a[:, rng.integers(0, n)] *= 10.0 ** rng.uniform(1, 6)
    elif law == 1:  # row scales over 2^+-20
        a *= (2.0 ** rng.uniform(-20, 20, (m, 1)))
    elif law == 2:  # column scales over 2^+-12
        a *= (2.0 ** rng.uniform(-12, 12, (1, n)))
    elif law == 3:  # sparse with exact zeros, a zero column now and then
        a *= rng.random((m, n)) < 0.35
        if rng.random() < 0.3:
            a[:, rng.integers(0, n)] = 0.0
    elif law == 4:  # integer-valued floats
        a = np.rint(a * rng.integers(1, 50)).astype(np.float64)
    elif law == 5:  # nearly rank one (massive cancellation in Ryser)
        a = np.outer(rng.uniform(0.5, 1.5, m), rng.uniform(0.5, 1.5, n)) + 1e-6 * a
    elif law == 6:  # tiny and huge magnitudes together
        a *= 10.0 ** rng.integers(-6, 7, (m, n))
    else:  # all positive, close to the ones matrix
        a = 1.0 + 1e-3 * a
    return a


def magsum2(a):
    return max(O.glynn_magnitude_sum(a), O.ryser_magnitude_sum(a, nthreads=1))


def test_harsh_float_laws():
    rng = np.random.default_rng(20261023)
    for case in range(int(os.environ.get("PERM_FUZZ_HARSH", "120"))):
        n = int(rng.integers(2, 17))
        m = int(rng.integers(1, n + 1)) if case % 2 else n
        a = harsh(rng, m, n, case % 8)
        if case % 5 == 4:
            a = a + 1j * harsh(rng, m, n, (case // 8) % 8)
        ref = O.dd_permanent("ryser" if m < n else "glynn", a, nthreads=4)
        M = magsum2(a)
        fns = [P.opt, P.glynn, P.ryser] + ([P.combinatoric] if math.perm(n, m) <= 500_000 else [])
        for fn in fns:
            got = fn(a)
            assert scaled_err(got, ref, M) <= TOL, (case, fn.__name__, m, n, case % 8, got, ref, M)


def test_harsh_integer_laws():
    rng = np.random.default_rng(20261024)
    for case in range(int(os.environ.get("PERM_FUZZ_HARSH", "120"))):
        n = int(rng.integers(2, 13))
        m = int(rng.integers(1, n + 1)) if case % 2 else n
        law = case % 4
        if law == 0:
            a = rng.integers(0, 3, (m, n))
            a[:, rng.integers(0, n)] *= int(rng.integers(1, 5000))
        elif law == 1:
            a = rng.integers(-3, 4, (m, n))
            a[rng.integers(0, m), :] *= int(rng.integers(1, 5000))
        elif law == 2:
            a = rng.integers(-50, 51, (m, n)) * (rng.random((m, n)) < 0.5)
        else:
            a = rng.integers(-1, 2, (m, n)) * int(10 ** rng.integers(0, 5))
        a = a.astype(np.int64)
        algs = ["glynn", "ryser"] + (["combinatoric"] if math.perm(n, m) <= 500_000 else [])
        for alg in algs:
            want, ovf = O.permanent(alg, a)
            fn = getattr(P, alg)
            if ovf:
                with pytest.raises(OverflowError):
                    fn(a)
            else:
                assert fn(a) == want, (case, alg, m, n, law)
        try:
            exact = O.exact_int128("ryser", a)
        except OverflowError:  # the permanent itself leaves int128 (the oracle refuses to wrap)
            exact = 1 << 127
        if abs(exact) < 1 << 90:
            for alg in algs:
                try:
                    got = getattr(P, alg)(a, exact="int128")
                except OverflowError:
                    # Glynn's raw sum carries 2^(n-1) (n-m)!: refusals only past the certified range
                    assert alg == "glynn" and abs(exact) * (1 << (n - 1)) * math.factorial(n - m) >= 1 << 126
                    continue
                assert got == exact, (case, alg, m, n, law)


def test_harsh_batches():
    """The batch entry points on the same laws: Laplace 8x8, set partitions
    (m <= 4 < n), thread- and warp-per-matrix Glynn / Ryser, segmented walks."""
    rng = np.random.default_rng(20261025)
    shapes = [(8, 8), (4, 10), (3, 7), (2, 12), (5, 5), (6, 9), (12, 12), (7, 14), (1, 6), (16, 16), (5, 8)]
    for case in range(int(os.environ.get("PERM_FUZZ_HARSH", "120")) // 4):
        m, n = shapes[case % len(shapes)]
        B = int(rng.integers(1, 200))
        cplx = case % 3 == 2
        A = np.stack([harsh(rng, m, n, (case + i) % 8) + (1j * harsh(rng, m, n, i % 8) if cplx else 0)
                      for i in range(B)])
        ref_alg = "combinatoric" if math.perm(n, m) <= 500_000 else ("ryser" if m < n else "glynn")
        picks = sorted(set(int(i) for i in rng.integers(0, B, 5)) | {0, B - 1})
        for bfn in (P.opt_batch, P.glynn_batch, P.ryser_batch):
            out = bfn(A)
            assert out.shape == (B,)
            for i in picks:
                r = O.dd_permanent(ref_alg if ref_alg != "combinatoric" else ("ryser" if m < n else "glynn"),
                                   A[i], nthreads=1)
                assert scaled_err(out[i], r, magsum2(A[i])) <= TOL, (case, bfn.__name__, m, n, i, out[i], r)


def test_harsh_medium_and_views():
    """15 <= n <= 22 on the harsh laws, from non-contiguous views, Fortran
    order, tall inputs (m > n) and strided CUDA tensors."""
    import torch

    rng = np.random.default_rng(20261026)
    for case in range(max(6, int(os.environ.get("PERM_FUZZ_HARSH", "120")) // 10)):
        n = int(rng.integers(15, 23))
        m = int(rng.integers(n - 5, n + 1))
        big = harsh(rng, 2 * m, 2 * n, case % 8)
        if case % 3 == 1:
            big = big + 1j * harsh(rng, 2 * m, 2 * n, (case + 3) % 8)
        view = big[::2, 1::2]  # strided, not contiguous
        a = np.ascontiguousarray(view)
        ref = O.dd_permanent("ryser" if m < n else "glynn", a, nthreads=16)
        M = magsum2(a)
        forms = {"view": view, "fortran": np.asfortranarray(a), "tall": a.T,
                 "cuda": torch.tensor(big, device="cuda")[::2, 1::2]}
        for name, x in forms.items():
            for fn in (P.opt, P.glynn, P.ryser):
                got = fn(x)
                assert scaled_err(got, ref, M) <= TOL, (case, name, fn.__name__, m, n, got, ref)


def test_full_size_laplace_expansions():
    """C5 (36x36 f64), C3a (24x24 c128) and C3b (20x28 c128, rectangular) at
    full size against their own Laplace expansion along a row: n minors, each
    an independent walk of one size less (for m < n the minor drops the row
    and one column).  A size-independent check that shares no walk with the
    value it checks; tolerance 1e-10 relative to sum_j |a_0j per(minor_j)|."""
    from paper_2510_03421_b200 import workloads as W

    for name, a in (("c5", W.c5(36)), ("c3a", W.c3a()), ("c3b", W.c3b())):
        m, n = a.shape
        per = P.glynn(a)
        rest = a[1:]
        terms = [a[0, j] * P.glynn(np.ascontiguousarray(np.delete(rest, j, axis=1))) for j in range(n)]
        lap = sum(terms)
        scale = sum(abs(t) for t in terms)
        assert abs(lap - per) <= TOL * scale, (name, per, lap, abs(lap - per) / scale)
