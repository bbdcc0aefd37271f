"""The two batch-only formulas of csrc/batch_bulk.cuh, restated in numpy and
checked against the oracle's restatement of the reference kernels (CPU):

* partition (m <= 6): per(A) = sum over set partitions pi of the rows of
  mu(pi) prod_{blocks b} p_b,  p_b = sum_j prod_{i in b} a_ij,
  mu(pi) = prod_b (-1)^(|b|-1) (|b|-1)!  -- Moebius inversion from "maps
  constant on blocks" to injective maps (the reference's combinatoric sum,
  src/_kernels.py:28-56, reorganised).
* row recursion (8x8, the engine's C2a kernel RowDp8Tm):
  f_L(S) = sum_{j in S} a_{L-1,j} f_{L-1}(S \\ {j}), per(A) = f_8({0..7}),
  with level 5 built by pushing the parked level 4 (first push a product).
* Laplace (8x8, the round-1 kernel, kept in tools/laplace8_variants.cuh):
  per(A) = sum_{|X|=4} per(A[0:4, X]) per(A[4:8, X^c]), the
  4x4 minors from 2x2 row-pair permanents q(P):
  per(H[:, X]) = sum_{P subset X, |P| = 2} q01(P) q23(X \\ P).

Also pins the symmetries the kernels rely on to read matrices without bank
conflicts (column rotation, row order inside a pair)."""
from __future__ import annotations

import itertools
import math

import numpy as np
import pytest

from oracle import oracle as O


def set_partitions(items):
    if not items:
        yield []
        return
    first, rest = items[0], items[1:]
    for p in set_partitions(rest):
        for i in range(len(p)):
            yield p[:i] + [[first] + p[i]] + p[i + 1:]
        yield [[first]] + p


def partition_formula(a):
    m, n = a.shape
    total = 0
    for pi in set_partitions(list(range(m))):
        term = 1
        for b in pi:
            term *= (-1) ** (len(b) - 1) * math.factorial(len(b) - 1)
            term *= np.prod(a[b, :], axis=0).sum()
        total += term
    return total


def laplace8(a):
    def q(r0, r1, i, k):
        return a[r0, i] * a[r1, k] + a[r0, k] * a[r1, i]

    def minor(rows, X):
        a_, b_, c_, d_ = X
        r0, r1, r2, r3 = rows
        splits = [((a_, b_), (c_, d_)), ((c_, d_), (a_, b_)), ((a_, c_), (b_, d_)), ((b_, d_), (a_, c_)),
                  ((a_, d_), (b_, c_)), ((b_, c_), (a_, d_))]
        return sum(q(r0, r1, *P) * q(r2, r3, *Q) for P, Q in splits)

    tot = 0.0
    for X in itertools.combinations(range(8), 4):
        Xc = tuple(j for j in range(8) if j not in X)
        tot += minor((0, 1, 2, 3), X) * minor((4, 5, 6, 7), Xc)
    return tot


def rowdp8(a):
    """The kernel's evaluation order: levels 2-4 and 6-8 pull, level 5 pushes
    level-4 entries in rank order (subsets ranked by increasing bit mask)."""
    n = a.shape[0]
    masks = {k: [m for m in range(1 << n) if bin(m).count("1") == k] for k in range(n + 1)}
    f = {1 << j: a[0, j] for j in range(n)}
    for L in range(2, n + 1):
        g = {}
        if L == 5:
            for T in masks[4]:
                for j in range(n):
                    if not (T >> j) & 1:
                        S = T | (1 << j)
                        g[S] = a[4, j] * f[T] if S not in g else g[S] + a[4, j] * f[T]
        else:
            for S in masks[L]:
                js = [j for j in range(n) if (S >> j) & 1]
                g[S] = sum(a[L - 1, j] * f[S & ~(1 << j)] for j in js)
        f = g
    return f[(1 << n) - 1]


def test_rowdp8_vs_oracle():
    rng = np.random.default_rng(18)
    for _ in range(3):
        ai = rng.integers(-2, 3, (8, 8)).astype(np.int64)
        assert rowdp8(ai) == O.permanent("glynn", ai)[0]  # exact on integers
    assert rowdp8(np.ones((8, 8))) == 40320.0
    assert rowdp8(np.eye(8)) == 1.0
    af = rng.standard_normal((8, 8)) / np.sqrt(8)
    ref = O.permanent("glynn", af)[0]
    assert abs(rowdp8(af) - ref) <= 1e-12 * O.glynn_magnitude_sum(af)
    # FP64 ops of the recursion, levels 2..8 (the kernel's 769 DFMA + 247 DMUL)
    assert sum(L * math.comb(8, L) for L in range(2, 9)) == 1016


def test_set_partition_counts():
    assert [sum(1 for _ in set_partitions(list(range(k)))) for k in range(1, 7)] == [1, 2, 5, 15, 52, 203]
    # |mu| summed over partitions of an m-set = m! (permutations by cycle type)
    for m in range(1, 6):
        s = sum(math.prod(math.factorial(len(b) - 1) for b in pi) for pi in set_partitions(list(range(m))))
        assert s == math.factorial(m)


@pytest.mark.parametrize("m,n", [(1, 1), (1, 5), (2, 2), (2, 7), (3, 3), (3, 8), (4, 4), (4, 10), (4, 13), (5, 7),
                                 (5, 10), (6, 8), (6, 9)])
def test_partition_formula_vs_oracle(m, n):
    rng = np.random.default_rng(100 * m + n)
    ai = rng.integers(-3, 4, (m, n)).astype(np.int64)
    assert partition_formula(ai) == O.permanent("combinatoric", ai)[0]  # exact on integers
    af = rng.standard_normal((m, n)) / np.sqrt(n)
    ref = O.permanent("combinatoric", af)[0]
    assert abs(partition_formula(af) - ref) <= 1e-12 * max(1.0, abs(ref))
    ac = af + 1j * rng.standard_normal((m, n))
    refc = O.permanent("ryser", ac)[0]
    assert abs(partition_formula(ac) - refc) <= 1e-11 * max(1.0, abs(refc))


def test_laplace8_vs_oracle():
    rng = np.random.default_rng(8)
    ai = rng.integers(-2, 3, (8, 8)).astype(np.int64)
    assert round(laplace8(ai.astype(np.float64))) == O.permanent("glynn", ai)[0]
    assert laplace8(np.ones((8, 8))) == 40320.0
    assert laplace8(np.eye(8)) == 1.0
    af = rng.standard_normal((8, 8)) / np.sqrt(8)
    ref = O.permanent("glynn", af)[0]
    assert abs(laplace8(af) - ref) <= 1e-12 * O.glynn_magnitude_sum(af)


def test_kernel_symmetries():
    """Laplace8Op reads its half with a column rotation by 2*rho (shared by
    both lanes of a matrix) and swaps the two rows of a 128-byte row when t:
    q01 / q23 are symmetric in their rows and per is column-permutation
    invariant.  PartitionOp rotates the row order (the combine is symmetric)."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal((8, 8))
    ref = laplace8(a)
    for rho in range(4):
        for t in (0, 1):
            b = np.roll(a, -2 * rho, axis=1)
            if t:
                b = b[[1, 0, 3, 2, 5, 4, 7, 6]]
            assert abs(laplace8(b) - ref) <= 1e-12 * max(1.0, abs(ref))
            assert abs(rowdp8(b) - ref) <= 1e-12 * max(1.0, abs(ref))
    r = rng.standard_normal((4, 10))
    for tau in range(4):
        assert abs(partition_formula(np.roll(r, -tau, axis=0)) - partition_formula(r)) <= 1e-12
