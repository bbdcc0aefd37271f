"""The FP32-quad exact int128 walk (csrc/int_walk32.cuh) against the oracle's
exact integer permanents and against the FP64-exact walk, bit for bit.
Needs a B200.

The walk is chosen by the host whenever the state entries group into quads
with bound products < 2^23 (engine_int.cu int_f32_quads); which kernel ran
is read from the est_kind slot of ``perm_walk_partial_i64``'s partial
(3 = FP32 estimate / integer upper levels, 4 = FP64 upper levels, 1 = the
FP64-exact walk of int_walk.cuh)."""
from __future__ import annotations

import json
import math
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2510_03421_b200 as P
from conftest import GOLDEN
from oracle import oracle as O
from paper_2510_03421_b200 import sharded as S
from paper_2510_03421_b200 import workloads as W

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def est_kind(alg, a):
    m, n = a.shape
    steps = 1 << (n - 1 if alg == "glynn" else n)
    return int(S.gpu_partial_int(alg, a, 0, steps, exact="int128")[5])


def cases():
    rng = np.random.default_rng(20251021)
    out = []
    # every quad count 3..5 (n = 9..18), odd and even, 0/1 and signed
    for n in (9, 10, 11, 12, 13, 15, 16, 17, 18):
        out.append(("01", rng.integers(0, 2, (n, n)).astype(np.int64)))
        out.append(("pm2", rng.integers(-2, 3, (n, n)).astype(np.int64)))
    return out


@pytest.mark.parametrize("alg", ["glynn", "ryser"])
def test_f32_walk_matches_oracle(alg):
    ran = set()
    for kind, a in cases():
        want = O.exact_int128(alg, a)
        assert getattr(P, alg)(a, exact="int128") == want, (kind, a.shape)
        ran.add(est_kind(alg, a))
    assert 4 in ran, ran  # the FP64-upper-level variant ran


def test_integer_upper_levels_variant():
    """Quads between 2^21 and 2^23: the four-quad products pass 2^84, so the
    96-bit products come from the integer multiplies (est_kind 3)."""
    rng = np.random.default_rng(5)
    kinds = set()
    for n in (14, 16):
        for _ in range(3):
            a = rng.integers(-5, 6, (n, n)).astype(np.int64)
            for alg in ("glynn", "ryser"):
                assert getattr(P, alg)(a, exact="int128") == O.exact_int128(alg, a), (alg, n)
                kinds.add(est_kind(alg, a))
    assert 3 in kinds, kinds


def test_large_entries_keep_the_fp64_exact_walk():
    """Column bounds past 2^23 / 4 per quad: not eligible, and still exact."""
    rng = np.random.default_rng(6)
    a = rng.integers(-300, 301, (12, 12)).astype(np.int64)
    assert est_kind("glynn", a) in (0, 1, 2)
    assert P.glynn(a, exact="int128") == O.exact_int128("glynn", a)


def test_rectangular_glynn_int128():
    """Ones-padded rectangular Glynn (pad rows flip too) through the quad walk."""
    rng = np.random.default_rng(8)
    for m, n in ((8, 12), (10, 13), (6, 16)):
        a = rng.integers(-2, 3, (m, n)).astype(np.int64)
        assert P.glynn(a, exact="int128") == O.exact_int128("glynn", a), (m, n)


def test_c4_configs_match_fixture_and_fp64_walk():
    """C4a / C4b through the quad walk equal the committed exact values; the
    FP64-exact walk (PERM_INT_F32=0, read at first use, so a subprocess) gives
    the same bits."""
    fix = json.load(open(GOLDEN / "c4.json"))
    a, b = W.c4a(), W.c4b()
    va, vb = P.glynn(a, exact="int128"), P.glynn(b, exact="int128")
    assert str(va) == fix["c4a_exact"] and str(vb) == fix["c4b_exact"]
    assert est_kind("glynn", a) == 4 and est_kind("glynn", b) in (3, 4)
    assert P.ryser(b, exact="int128") == vb
    code = ("import sys; sys.path.insert(0, '.'); import paper_2510_03421_b200 as P; "
            "from paper_2510_03421_b200 import workloads as W; "
            "print(P.glynn(W.c4b(), exact='int128'))")
    env = dict(os.environ, PERM_INT_F32="0")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert int(r.stdout.strip().splitlines()[-1]) == vb


def test_sharded_ranges_sum_to_the_whole():
    """Unaligned shard boundaries (world 3) through the partial / finish protocol."""
    a = W.c4b()[:20, :20].copy()
    want = O.exact_int128("glynn", a)
    assert S.sharded_permanent(a, alg="glynn", exact="int128") == want
    m, n = a.shape
    for alg in ("glynn", "ryser"):
        parts = [S.gpu_partial_int(alg, a, *S.shard_range(alg, m, n, r, 3), exact="int128") for r in range(3)]
        assert {int(p[5]) for p in parts} <= {3, 4}
        assert S.finish_int(alg, a, np.stack(parts), exact="int128") == want


def test_int128_fuzz():
    """Seeded fuzz of the exact int128 entry points over shapes 9 <= n <= 22
    (square and rectangular Glynn, square Ryser), 0/1 densities and signed
    entry ranges on both sides of the quad walk's eligibility bounds, against
    the oracle's exact integers.  PERM_FUZZ_INT128 cases (default 80)."""
    rng = np.random.default_rng(20261022)
    kinds = {}
    for case in range(int(os.environ.get("PERM_FUZZ_INT128", "80"))):
        n = int(rng.integers(9, 23))
        m = n if case % 3 else int(rng.integers(max(2, n - 6), n + 1))
        law = case % 5
        if law == 0:
            a = (rng.random((m, n)) < rng.uniform(0.2, 0.9)).astype(np.int64)
        elif law == 1:
            k = int(rng.integers(1, 4))
            a = rng.integers(-k, k + 1, (m, n)).astype(np.int64)
        elif law == 2:
            k = int(rng.integers(4, 13))
            a = rng.integers(-k, k + 1, (m, n)).astype(np.int64)
        elif law == 3:
            a = ((rng.random((m, n)) < 0.3) * rng.integers(-40, 41, (m, n))).astype(np.int64)
        else:
            a = rng.integers(0, 3, (m, n)).astype(np.int64)
            a[:, int(rng.integers(0, n))] *= int(rng.integers(1, 2000))  # one heavy column
        # the oracle's int128 walks wrap silently: Ryser's raw sum is the
        # permanent itself, so it is the reference value (|per| < 2^127 here)
        try:
            want = O.exact_int128("ryser", a)
        except OverflowError:  # the permanent itself is past int128 (the oracle refuses to wrap)
            continue
        for alg in ("glynn",) + (("ryser",) if m == n else ()):
            try:
                got = getattr(P, alg)(a, exact="int128")
            except OverflowError:
                # allowed only when the walk's raw sum (value x 2^(n-1) (n-m)!
                # for Glynn) is past the certified range |raw| < 2^126
                raw = abs(want) * ((1 << (n - 1)) * math.factorial(n - m) if alg == "glynn" else 1)
                assert raw >= 1 << 126, (case, alg, m, n, want)
                continue
            assert got == want, (case, alg, m, n, law)
            k = est_kind(alg, a) if m == n else -1
            kinds[k] = kinds.get(k, 0) + 1
    assert kinds.get(4, 0) > 0 and kinds.get(3, 0) + kinds.get(1, 0) + kinds.get(2, 0) + kinds.get(0, 0) > 0, kinds


def test_rectangular_glynn_small_integers_stay_exact():
    """Regression (found by the fuzz above): a small rectangular integer matrix
    with one heavy column once took the certified float route, whose power-of-
    two pre-scale makes the rectangular Glynn products inexact (84 off)."""
    a = np.array([[2, 0, 0, 0, 2, 0, 0, 674, 0], [0, 2, 0, 1, 2, 2, 2, 0, 2], [2, 1, 2, 1, 2, 1, 1, 674, 1],
                  [0, 0, 0, 0, 1, 1, 0, 674, 1], [2, 2, 2, 2, 1, 0, 1, 337, 1], [1, 2, 0, 2, 0, 0, 0, 0, 2],
                  [2, 1, 1, 0, 2, 0, 0, 337, 2]], dtype=np.int64)
    want = O.permanent("combinatoric", a)[0]
    assert want == 32535348
    assert P.glynn(a, exact="int128") == want
    assert P.glynn(a) == want and P.ryser(a) == want and P.combinatoric(a) == want and P.opt(a) == want
    rng = np.random.default_rng(77)
    for _ in range(40):  # small rectangular integer matrices, default (checked) and int128
        n = int(rng.integers(3, 11))
        m = int(rng.integers(1, n))
        b = rng.integers(0, 3, (m, n)).astype(np.int64)
        b[:, int(rng.integers(0, n))] *= int(rng.integers(1, 3000))
        ref, ovf = O.permanent("glynn", b)
        if not ovf:
            assert P.glynn(b) == ref, b
        assert P.glynn(b, exact="int128") == O.exact_int128("ryser", b), b


def test_c4_full_size_properties():
    """C4a / C4b at full size through size-independent properties of the
    permanent, all exact integers: Laplace expansion along a row (n minors of
    size n - 1, each its own exact walk), invariance under row / column
    permutations and transposition, multilinearity in a row."""
    rng = np.random.default_rng(4)
    for a in (W.c4a(), W.c4b()):
        n = a.shape[0]
        per = P.glynn(a, exact="int128")
        row = int(rng.integers(0, n))
        rest = np.delete(a, row, axis=0)
        lap = 0
        for j in range(n):
            if a[row, j]:
                lap += int(a[row, j]) * P.glynn(np.ascontiguousarray(np.delete(rest, j, axis=1)), exact="int128")
        assert lap == per
        pr, pc = rng.permutation(n), rng.permutation(n)
        assert P.glynn(np.ascontiguousarray(a[pr][:, pc]), exact="int128") == per
        assert P.glynn(np.ascontiguousarray(a.T), exact="int128") == per
        b = a.copy()
        b[row] *= 3
        assert P.glynn(b, exact="int128") == 3 * per
        c = a.copy()
        c[row] = rng.integers(0, 2, n)
        d = a.copy()
        d[row] = a[row] + c[row]
        assert P.glynn(d, exact="int128") == per + P.glynn(c, exact="int128")
