"""The three exact algorithms in square and rectangular form, on the GPU.

Mirror of the reference's ``permanent.algorithms``
(/root/reference/pkg/src/permanent/algorithms.py, "src/algorithms.py"):
same names, shape contracts (ValueError), step budget
(``StepBudgetExceeded``) and result types.  Integer matrices keep the
reference's checked-int64 semantics by default: ``overflowed`` is set exactly
when the reference's kernels would report it (the engine replays the
reference's checks in parallel).  ``exact="int128"`` opts into the certified
exact path (value = exact Python int, overflowed = "does not fit int64",
the convention of src/reference.py:136-156).

``compiled`` is accepted for signature compatibility (src/algorithms.py:55-58
switches between interpreted and numba kernels); there is one CUDA path and
no CPU fallback.
"""
from __future__ import annotations

import enum
import math

from . import engine
from .core import ElementKind, Matrix, PermanentResult


class AlgorithmId(enum.Enum):
    """Algorithms known to dispatch, tuner and CLI (src/algorithms.py:26-31)."""

    COMBINATORIC = "combinatoric"
    RYSER = "ryser"
    GLYNN = "glynn"


class StepBudgetExceeded(RuntimeError):
    """The combinatoric enumeration is larger than the configured budget."""


#: src/algorithms.py:40 -- combinatoric runs above this many permutations are refused
DEFAULT_STEP_BUDGET = 2_000_000_000
#: src/algorithms.py:44 -- kept for API compatibility (no interpreted mode here)
COMPILE_STEP_THRESHOLD = 20_000
#: src/algorithms.py:47 -- Gray-walk counters cap the walks at 62 columns
_MAX_ENUM_COLS = 62

_EXACT_MODES = (None, "int64", "int128")


def _need(cond: bool, msg: str):
    if not cond:
        raise ValueError(msg)


def _float_result(value, kind: ElementKind) -> PermanentResult:
    return PermanentResult(float(value) if kind is ElementKind.FLOAT64 else complex(value))


def _int_walk(alg: str, a: Matrix, exact) -> PermanentResult:
    if exact not in _EXACT_MODES:
        raise ValueError(f"exact must be one of {_EXACT_MODES}, got {exact!r}")
    width = 128 if exact == "int128" else 64
    value, flag = engine.exact_int(alg, a.data, width=width)
    return PermanentResult(int(value), bool(flag))


def permanent_combinatoric(a: Matrix, step_budget: int = DEFAULT_STEP_BUDGET,
                           compiled=None, exact=None) -> PermanentResult:
    """Sum over all m-permutations of the columns (src/algorithms.py:71-90).
    Integer matrices: checked int64 by default, ``exact="int128"`` for the
    exact int128 DFS (a-priori certified)."""
    _need(a.m <= a.n, f"need m <= n, got {a.m}x{a.n}; transpose first")
    if exact not in _EXACT_MODES:
        raise ValueError(f"exact must be one of {_EXACT_MODES}, got {exact!r}")
    perms = math.perm(a.n, a.m)
    if perms > step_budget:
        raise StepBudgetExceeded(
            f"combinatoric on {a.m}x{a.n} needs {perms} permutations (> budget {step_budget})")
    value, ovf, _ = engine.comb(a.data, step_budget, width=128 if exact == "int128" else 64)
    if a.kind is ElementKind.INT64:
        return PermanentResult(int(value), bool(ovf))
    return _float_result(value, a.kind)


def permanent_ryser_square(a: Matrix, compiled=None, exact=None) -> PermanentResult:
    """Inclusion-exclusion over column subsets, square only (src/algorithms.py:93-107)."""
    _need(a.m == a.n, f"square form needs m == n, got {a.m}x{a.n}")
    _need(a.n <= _MAX_ENUM_COLS, f"subset walk over {a.n} columns exceeds 2^62 steps")
    if a.kind is ElementKind.INT64:
        return _int_walk("ryser", a, exact)
    return _float_result(engine.walk("ryser", a.data)[0], a.kind)


#: columns of the combination-ordered kernels (csrc/comb.cuh kCombMaxN); the
#: reference's ryser_rect and combinatoric have no column cap
_MAX_COMB_COLS = 256


def permanent_ryser_rectangular(a: Matrix, compiled=None, exact=None) -> PermanentResult:
    """Binomial-weighted Ryser for m <= n, square included (src/algorithms.py:118-137).

    Integers keep the reference's checked-int64 semantics of ryser_rect_int:
    the lexicographic combination order runs for every m <= n (the square
    Gray walk of ``permanent_ryser_square`` checks other intermediates, so
    its overflow flag could differ near the int64 onset).  Floats take the
    popcount-weighted Gray walk up to 62 columns (or the combination order
    where it is cheaper), and the combination order past 62 columns."""
    _need(a.m <= a.n, f"need m <= n, got {a.m}x{a.n}; transpose first")
    _need(a.m <= _MAX_ENUM_COLS and a.n <= _MAX_COMB_COLS,
          f"rectangular Ryser supports m <= {_MAX_ENUM_COLS}, n <= {_MAX_COMB_COLS}; got {a.m}x{a.n}")
    if a.kind is ElementKind.INT64:
        if exact == "int128" and a.n <= _MAX_ENUM_COLS:
            return _int_walk("ryser", a, exact)
        if exact not in _EXACT_MODES:
            raise ValueError(f"exact must be one of {_EXACT_MODES}, got {exact!r}")
        value, ovf = engine.ryser_rect(a.data)
        return PermanentResult(int(value), bool(ovf))
    if a.n > _MAX_ENUM_COLS:
        return _float_result(engine.ryser_rect(a.data)[0], a.kind)
    return _float_result(engine.walk("ryser", a.data)[0], a.kind)


def permanent_glynn_square(a: Matrix, compiled=None, exact=None) -> PermanentResult:
    """Sign-vector (Glynn) form over 2^(n-1) Gray-ordered vectors (src/algorithms.py:140-160)."""
    _need(a.m == a.n, f"square form needs m == n, got {a.m}x{a.n}")
    _need(a.n <= _MAX_ENUM_COLS, f"sign walk over {a.n} columns exceeds 2^61 steps")
    if a.kind is ElementKind.INT64:
        return _int_walk("glynn", a, exact)
    return _float_result(engine.walk("glynn", a.data)[0], a.kind)


def permanent_glynn_rectangular(a: Matrix, compiled=None, exact=None) -> PermanentResult:
    """Glynn for m < n via virtual all-ones rows (src/algorithms.py:163-184),
    with the real rows pre-scaled by a power of two on the GPU (exact
    algebra; fixes the padding's cancellation)."""
    _need(a.m < a.n, f"rectangular form needs m < n, got {a.m}x{a.n}")
    _need(a.n <= _MAX_ENUM_COLS, f"sign walk over {a.n} columns exceeds 2^61 steps")
    if a.kind is ElementKind.INT64:
        return _int_walk("glynn", a, exact)
    return _float_result(engine.walk("glynn", a.data)[0], a.kind)


def run_algorithm(a: Matrix, alg: AlgorithmId, compiled=None,
                  step_budget: int = DEFAULT_STEP_BUDGET, exact=None) -> PermanentResult:
    """One algorithm on an m <= n matrix, square or rectangular form by shape
    (src/algorithms.py:187-201)."""
    if alg is AlgorithmId.COMBINATORIC:
        return permanent_combinatoric(a, step_budget=step_budget, compiled=compiled, exact=exact)
    if alg is AlgorithmId.RYSER:
        if a.m == a.n:
            return permanent_ryser_square(a, compiled=compiled, exact=exact)
        return permanent_ryser_rectangular(a, compiled=compiled, exact=exact)
    if alg is AlgorithmId.GLYNN:
        if a.m == a.n:
            return permanent_glynn_square(a, compiled=compiled, exact=exact)
        return permanent_glynn_rectangular(a, compiled=compiled, exact=exact)
    raise ValueError(f"unknown algorithm {alg!r}")


def permanent_with_magsum(a: Matrix, alg: AlgorithmId):
    """(value, M): the float permanent and its magnitude sum M = normalized
    sum of |terms| of the Glynn / Ryser walk -- the scale of the parity
    metric."""
    _need(a.kind is not ElementKind.INT64, "magnitude sums are defined for float inputs")
    _need(a.m <= a.n, "need m <= n")
    name = "glynn" if alg is AlgorithmId.GLYNN else "ryser"
    v, mg = engine.walk(name, a.data, magsum=True)
    return (float(v) if a.kind is ElementKind.FLOAT64 else complex(v)), mg
