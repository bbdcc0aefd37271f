"""Seeded synthetic inputs for the BASELINE.json configurations.

No public dataset is involved; every config is a seeded draw with the shape
and value distribution BASELINE.json names.  Seeds follow SURVEY 8(d):
``np.random.default_rng([2510, 3421, k])``; for the "/sqrt(n)" scalings n is
the number of columns.
"""
from __future__ import annotations

import math

import numpy as np


def rng(k: int) -> np.random.Generator:
    return np.random.default_rng([2510, 3421, k])


def c1(batch: int = 64) -> np.ndarray:
    """C1: 64 float64 12x12, iid U[-1,1]."""
    return rng(1).uniform(-1.0, 1.0, (batch, 12, 12))


def c2a(batch: int = 1_000_000) -> np.ndarray:
    """C2a: float64 8x8, iid N(0,1)/sqrt(8)."""
    return rng(2).standard_normal((batch, 8, 8)) / math.sqrt(8)


def c2b(batch: int = 1_000_000) -> np.ndarray:
    """C2b: float64 4x10, iid N(0,1)/sqrt(10)."""
    return rng(3).standard_normal((batch, 4, 10)) / math.sqrt(10)


def c3a() -> np.ndarray:
    """C3a: complex128 24x24, re/im iid U[-1,1]/sqrt(24) (real part drawn first)."""
    g = rng(4)
    re = g.uniform(-1.0, 1.0, (24, 24))
    im = g.uniform(-1.0, 1.0, (24, 24))
    return (re + 1j * im) / math.sqrt(24)


def c3b() -> np.ndarray:
    """C3b: complex128 20x28, same law, /sqrt(28)."""
    g = rng(5)
    re = g.uniform(-1.0, 1.0, (20, 28))
    im = g.uniform(-1.0, 1.0, (20, 28))
    return (re + 1j * im) / math.sqrt(28)


def bernoulli01(n: int, g: np.random.Generator) -> np.ndarray:
    """0/1 Bernoulli(0.5) n x n, redrawn until every row and column is nonzero."""
    while True:
        a = (g.random((n, n)) < 0.5).astype(np.int64)
        if a.sum(axis=0).min() > 0 and a.sum(axis=1).min() > 0:
            return a


def c4a(n: int = 32) -> np.ndarray:
    """C4a: 0/1 32x32 Bernoulli(0.5), every row and column nonzero."""
    return bernoulli01(n, rng(6))


def c4b(n: int = 28) -> np.ndarray:
    """C4b: int64 28x28 uniform in {-2..2}."""
    return rng(7).integers(-2, 3, (n, n)).astype(np.int64)


def c5(n: int = 36) -> np.ndarray:
    """C5: float64 36x36 iid U[0,1]/36 (n-sweep: seed 10+n)."""
    k = 8 if n == 36 else 10 + n
    return rng(k).uniform(0.0, 1.0, (n, n)) / n


def rank_one(n: int = 36):
    """u v^T with u, v ~ U[0.9, 1.1] (k=9); per = n! * prod(u) * prod(v)."""
    g = rng(9)
    u = g.uniform(0.9, 1.1, n)
    v = g.uniform(0.9, 1.1, n)
    exact = math.factorial(n) * float(np.prod(u)) * float(np.prod(v))
    return np.outer(u, v), exact


def ones(n: int = 36):
    """J_n; per = n!."""
    return np.ones((n, n)), float(math.factorial(n))
