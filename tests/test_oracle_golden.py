"""Pin the CPU oracle (oracle/perm_oracle.c) to the reference: its literal
restatements must reproduce the reference's golden vectors bit for bit, and
its higher-precision / exact walks must agree with them.  CPU only."""
from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import decode_matrix, decode_value, parity_case
from oracle import oracle as O


def test_parity_json_bitwise(parity_cases):
    """All 300 reference golden vectors (pkg/frontend/tests/fixtures/parity.json)."""
    assert len(parity_cases) == 300
    for c in parity_cases:
        a, alg, exp = parity_case(c)
        mat = a if a.shape[0] <= a.shape[1] else a.T
        alg_ = "glynn" if alg == "opt" else alg
        if alg == "opt":
            # the reference's default dispatch (src/dispatch.py:84-95)
            from paper_2510_03421_b200.dispatch import default_params, select_algorithm

            alg_ = select_algorithm(mat.shape[0], mat.shape[1], default_params()).value
        value, ovf = O.permanent(alg_, mat)
        assert not ovf
        if isinstance(exp, int):
            assert value == exp
        else:
            assert value == exp, (alg, a.shape, value, exp)  # bit-exact


def test_reference_cases_bitwise(ref_cases):
    """Every algorithm, every kind, m <= n <= 9, incl. int overflow KATs."""
    n_checked = 0
    for case in ref_cases:
        a = decode_matrix(case["matrix"])
        for alg, r in case["results"].items():
            exp = decode_value(r["value"])
            value, ovf = O.permanent(alg, a, compiled=True)  # fixtures ran compiled
            assert ovf == r["overflowed"], (alg, a)
            if not ovf:
                if isinstance(exp, float) and math.isnan(exp):
                    assert math.isnan(value)
                else:
                    assert value == exp, (alg, a.shape, value, exp)
            n_checked += 1
    assert n_checked > 900


def test_reference_int_walk_near_overflow(ref_int_walk):
    """Checked-int64 flags near the overflow onset and the
    int128 oracle's exact values."""
    for case in ref_int_walk:
        a = decode_matrix(case["matrix"])
        exact = int(case["exact"])
        for alg, r in case["results"].items():
            value, ovf = O.permanent(alg, a)
            assert ovf == r["overflowed"]
            if not ovf:
                assert value == decode_value(r["value"]) == exact
        assert O.exact_int128("ryser", a) == exact


def test_int128_walk_matches_bruteforce(rng):
    for n in range(1, 8):
        for m in range(1, n + 1):
            a = rng.integers(-5, 6, (m, n)).astype(np.int64)
            exact = O.brute_force(a.tolist())
            assert O.exact_int128("glynn", a) == exact
            assert O.exact_int128("ryser", a) == exact


def test_dd_walk_matches_literal(rng):
    for n in (3, 6, 9, 12):
        for m in (n, max(1, n - 2)):
            a = rng.uniform(-1, 1, (m, n))
            ref = O.permanent("ryser", a)[0]
            for alg in ("glynn", "ryser"):
                v = O.dd_permanent(alg, a, nthreads=2)
                assert abs(v - ref) <= 1e-11 * max(abs(ref), O.glynn_magnitude_sum(a))
            c = a + 1j * rng.uniform(-1, 1, (m, n))
            ref = O.permanent("ryser", c)[0]
            v = O.dd_permanent("glynn", c, nthreads=2)
            assert abs(v - ref) <= 1e-11 * max(abs(ref), O.glynn_magnitude_sum(c))


def test_range_walk_sharding_identity(rng):
    """Sum over contiguous Gray ranges = the whole walk."""
    a = rng.integers(-3, 4, (9, 9)).astype(np.int64)
    s = O.walk_setup("glynn", a)
    whole = O.walk_i128_mt(s, nthreads=1)
    parts = sum(O.walk_i128_mt(s, k0, k1, nthreads=1)
                for k0, k1 in ((0, 37), (37, 100), (100, 256)))
    assert parts == whole
    assert whole // 2 ** 8 == O.brute_force(a.tolist())


def test_closed_forms():
    from paper_2510_03421_b200 import workloads as W

    for n in (8, 10):
        a, exact = W.ones(n)
        assert O.dd_permanent("glynn", a, nthreads=2) == pytest.approx(exact, rel=1e-14)
    u = np.linspace(0.9, 1.1, 9)
    v = np.linspace(1.1, 0.95, 9)
    exact = math.factorial(9) * np.prod(u) * np.prod(v)
    assert O.dd_permanent("glynn", np.outer(u, v), nthreads=2) == pytest.approx(exact, rel=1e-13)


def test_prescaled_rect_glynn_is_well_conditioned(rng):
    """power-of-two pre-scaling of the real rows fixes the
    all-ones padding's cancellation (here in the oracle's dd walk)."""
    a = (rng.uniform(-1, 1, (6, 13)) + 1j * rng.uniform(-1, 1, (6, 13))) / 4.0
    ref = O.permanent("combinatoric", a)[0]
    v = O.dd_permanent("glynn", a, nthreads=4)
    assert abs(v - ref) <= 1e-12 * abs(ref)


def test_magnitude_sum_two_restatements_agree(rng):
    """The scale M of metric (ii) has two oracle restatements: the numpy
    brute walk (n <= 14) and the C double-double walk's |term| sum (used
    above 14 columns).  They agree to 1e-13 on square, rectangular and
    complex shapes, so the GPU tests' M pin (test_gpu_parity.py
    test_engine_magsum_pinned_to_oracle) is anchored in both."""
    shapes = [(12, 12, False), (9, 14, True), (5, 13, False), (14, 14, True), (1, 6, False)]
    for m, n, cplx in shapes:
        a = rng.uniform(-1, 1, (m, n)) + (1j * rng.uniform(-1, 1, (m, n)) if cplx else 0)
        brute = O.glynn_magnitude_sum(a)
        sc = O.prescale_factor(a) if m < n else 1.0
        _, _, mg = O.walk_dd_mt(O.walk_setup("glynn", a, scale=sc), nthreads=2, mag=True)
        viac = mg / (2.0 ** (n - 1) * math.factorial(n - m) * sc ** m)
        assert abs(brute - viac) <= 1e-13 * brute, (m, n, cplx, brute, viac)


def test_wide_column_forms(rng):
    """Past 62 columns (no cap in the reference's combinatoric / ryser_rect):
    the oracle's DFS and combination-order Ryser agree with brute force."""
    for m, n in ((1, 200), (2, 90), (3, 70)):
        a = rng.integers(-3, 4, (m, n)).astype(np.int64)
        exact = O.brute_force(a.tolist())
        assert O.permanent("combinatoric", a) == (exact, False)
        assert O.kernel("ryser_rect", a) == (exact, False)
        f = a.astype(np.float64)
        assert O.permanent("combinatoric", f)[0] == exact
