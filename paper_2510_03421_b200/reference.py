"""``permanent_reference``: the reference package's structural oracle entry
point (/root/reference/pkg/src/permanent/reference.py:136-156), exported by
its public API, served here by the engine's exact / extended-precision walks.

Semantics kept: m <= n required (ValueError), guarded to n <= 20
(StepBudgetExceeded), integer results exact at any size with
``overflowed`` meaning "the value lies outside int64" (not an arithmetic
failure).  The reference evaluates naive transcriptions in Python big ints;
here integers come from the certified int128 walk and floats from the
double-double GPU walk, so the values are exact / correctly
rounded rather than naive-order floats.
"""
from __future__ import annotations

from .algorithms import AlgorithmId, StepBudgetExceeded
from .core import INT64_MAX, INT64_MIN, ElementKind, Matrix, PermanentResult

MAX_REFERENCE_COLS = 20


def permanent_reference(a: Matrix, alg: AlgorithmId) -> PermanentResult:
    from . import engine
    from .algorithms import run_algorithm

    if a.m > a.n:
        raise ValueError(f"need m <= n, got {a.m}x{a.n}; transpose first")
    if a.n > MAX_REFERENCE_COLS:
        raise StepBudgetExceeded(f"reference implementations are guarded to n <= {MAX_REFERENCE_COLS}")
    if not isinstance(alg, AlgorithmId):
        raise ValueError(f"unknown algorithm {alg!r}")
    if a.kind is ElementKind.INT64:
        value = run_algorithm(a, AlgorithmId.RYSER if alg is AlgorithmId.COMBINATORIC else alg,
                              exact="int128").value
        return PermanentResult(int(value), not (INT64_MIN <= value <= INT64_MAX))
    name = "glynn" if alg is AlgorithmId.GLYNN else "ryser"
    (rh, rl), (ih, il) = engine.walk_dd(name, a.data)
    if a.kind is ElementKind.FLOAT64:
        return PermanentResult(rh + rl)
    return PermanentResult(complex(rh + rl, ih + il))
