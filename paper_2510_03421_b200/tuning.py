"""Tuning file v1 (line-oriented key=value) and the B200 crossover tuner.

File format: the reference's (/root/reference/pkg/src/permanent/tuner.py:340-383):
``format_version=1``, ``source``, ``host``, ``created_at`` and ``p1``..``p8``,
one key per line, floats in shortest round-trip form; unknown, duplicate or
missing keys and other versions are rejected with ValueError.

Two fits over B200 kernel timings {(m, n): {alg: seconds}}:
* ``run_tuning`` -- the reference's procedure (tuner.py:96-333, same names:
  ``algorithm_feasible``, ``time_algorithm``, ``build_label_grid``,
  ``fit_hard_margin_svm``, ``plane_intersection``, ``assemble_params``):
  timing grid, labels with margin ratios, near-tie filter, two
  maximum-margin lines over (r, n) (``svm.py``; weighted minimum-cost
  fallback when the labels are not separable), p4 from the square cutoff,
  p8 from the lines' crossing;
* ``fit_params`` -- a direct search minimizing the summed relative slowdown
  (GPU timings below ~50 us are launch-overhead dominated, so labels there
  are noisy and rarely separable; profiles/r2_dispatch_fit.txt compares the
  two on the same B200 timings).
"""
from __future__ import annotations

import datetime
import itertools
import math
import platform
from pathlib import Path

from .dispatch import TuningParams

_KEYS = ("format_version", "source", "host", "created_at",
         "p1", "p2", "p3", "p4", "p5", "p6", "p7", "p8")


def emit_tuning_file(params: TuningParams, path) -> None:
    """Write ``params`` as a version-1 tuning file."""
    out = [f"format_version=1", f"source={params.source}", f"host={params.host}",
           f"created_at={params.created_at}"]
    out += [f"p{k}={getattr(params, f'p{k}')!r}" for k in range(1, 9)]
    Path(path).write_text("\n".join(out) + "\n", encoding="utf-8")


def load_tuning_file(path) -> TuningParams:
    """Parse and validate a version-1 tuning file."""
    fields: dict[str, str] = {}
    for no, raw in enumerate(Path(path).read_text(encoding="utf-8").splitlines(), start=1):
        line = raw.strip()
        if not line:
            continue
        key, sep, value = line.partition("=")
        if not sep:
            raise ValueError(f"{path}:{no}: expected key=value, got {line!r}")
        if key not in _KEYS:
            raise ValueError(f"{path}:{no}: unknown key {key!r}")
        if key in fields:
            raise ValueError(f"{path}:{no}: duplicate key {key!r}")
        fields[key] = value
    missing = [k for k in _KEYS if k not in fields]
    if missing:
        raise ValueError(f"{path}: missing required key {missing[0]!r}")
    if fields["format_version"] != "1":
        raise ValueError(f"{path}: unsupported format_version {fields['format_version']!r}")
    ps = {f"p{k}": float(fields[f"p{k}"]) for k in range(1, 9)}
    return TuningParams(**ps, source=fields["source"], created_at=fields["created_at"],
                        host=fields["host"])


# ---------------------------------------------------------------------------
# B200 crossover tuner
# ---------------------------------------------------------------------------

def _select(params, m, n):
    from .dispatch import select_algorithm

    return select_algorithm(m, n, params).value


def _regret_line(cells: dict, pos: str, neg: str, skip):
    """Line (a, b, c) with a r + b n + c > 0 -> `pos`, else `neg`, minimizing
    the summed slowdown over `cells` ({(m, n): {alg: s}}); None if degenerate."""
    X, y, w = [], [], []
    for k, t in cells.items():
        if skip(k) or pos not in t or neg not in t:
            continue
        best = min(t.values())
        ca, cb = t[pos] / best - 1.0, t[neg] / best - 1.0
        X.append([k[0] / k[1], k[1]])
        y.append(1.0 if ca < cb else -1.0)
        w.append(abs(ca - cb))
    if len(X) < 2 or len(set(y)) < 2:
        return None
    from . import svm

    wv, b, _ = svm.min_misclassification_plane(np.array(X, float), np.array(y), angles=720, weights=np.array(w))
    if wv[0] == 0 and wv[1] == 0:
        return None
    return float(wv[0]), float(wv[1]), float(b)


def _penalty(slowdown: float) -> float:
    """Regret of one cell: the slowdown over the fastest, plus a hinge above
    1.15x, so the fit keeps a margin under the 1.25x acceptance bar where
    per-call timings jitter by ~10% (microsecond calls on the GPU box)."""
    return (slowdown - 1.0) + 4.0 * max(0.0, slowdown - 1.15)


def fit_params(timings: dict, host: str = "") -> TuningParams:
    """Fit p1..p8 to measured timings {(m, n): {alg: seconds}} by minimizing
    the summed relative slowdown of the selected algorithm (grid search)."""
    cells = {k: v for k, v in timings.items() if v}

    def cost(p):
        tot = 0.0
        for (m, n), t in cells.items():
            best = min(t.values())
            pick = _select(p, m, n)
            tot += _penalty(t[pick] / best) if pick in t else 1e6
        return tot

    best_p, best_c = None, math.inf
    slopes = (-2.0, -1.0, -0.5, 0.5, 1.0, 2.0)
    nslopes = (-0.2, -0.1, -0.05, -0.02, 0.0, 0.02, 0.05, 0.1)
    for p8 in range(4, 21):
        for p4 in range(2, min(p8, 9) + 1):
            # regime lines: coarse search of (p1, p2, p3), then (p5, p6, p7)
            base = TuningParams(p1=-1.0, p2=-0.1, p3=1.0, p4=float(p4), p5=1.0, p6=0.0, p7=-0.5,
                                p8=float(p8), source="machine-tuned")
            cand1 = []
            for p1, p2 in itertools.product(slopes, nslopes):
                if p1 == 0 and p2 == 0:
                    continue
                for p3 in (-2.0, -1.0, -0.5, 0.0, 0.5, 1.0, 1.5, 2.0, 3.0):
                    cand1.append((p1, p2, p3))
            small = {k: v for k, v in cells.items() if k[1] <= p8}
            large = {k: v for k, v in cells.items() if k[1] > p8}

            def sub_cost(p, subset):
                tot = 0.0
                for (m, n), t in subset.items():
                    pick = _select(p, m, n)
                    tot += _penalty(t[pick] / min(t.values())) if pick in t else 1e6
                return tot

            b1, c1 = None, math.inf
            for p1, p2, p3 in cand1:
                p = TuningParams(p1=p1, p2=p2, p3=p3, p4=float(p4), p5=1.0, p6=0.0, p7=-0.5,
                                 p8=float(p8), source="machine-tuned")
                c = sub_cost(p, small)
                if c < c1:
                    b1, c1 = (p1, p2, p3), c
            b2, c2 = None, math.inf
            for p5, p6 in itertools.product(slopes, nslopes):
                if p5 == 0 and p6 == 0:
                    continue
                for p7 in (-3.0, -2.0, -1.0, -0.5, -0.25, 0.0, 0.25, 0.5, 1.0, 2.0):
                    p = TuningParams(p1=b1[0], p2=b1[1], p3=b1[2], p4=float(p4), p5=p5, p6=p6, p7=p7,
                                     p8=float(p8), source="machine-tuned")
                    c = sub_cost(p, large)
                    if c < c2:
                        b2, c2 = (p5, p6, p7), c
            # refine each regime line with the weighted min-cost line search:
            # for a two-way choice, the total slowdown is the regret-weighted
            # misclassification count (weight |cost_a - cost_b|)
            r1 = _regret_line(small, "combinatoric", "glynn", lambda k: k[0] == k[1] and k[1] <= p4)
            if r1 is not None:
                p = TuningParams(p1=r1[0], p2=r1[1], p3=r1[2], p4=float(p4), p5=1.0, p6=0.0, p7=-0.5,
                                 p8=float(p8), source="machine-tuned")
                c = sub_cost(p, small)
                if c < c1:
                    b1, c1 = r1, c
            r2 = _regret_line(large, "glynn", "ryser", lambda k: False)
            if r2 is not None:
                p = TuningParams(p1=b1[0], p2=b1[1], p3=b1[2], p4=float(p4), p5=r2[0], p6=r2[1], p7=r2[2],
                                 p8=float(p8), source="machine-tuned")
                c = sub_cost(p, large)
                if c < c2:
                    b2, c2 = r2, c
            if c1 + c2 < best_c:
                best_c = c1 + c2
                best_p = TuningParams(p1=b1[0], p2=b1[1], p3=b1[2], p4=float(p4), p5=b2[0], p6=b2[1],
                                      p7=b2[2], p8=float(p8), source="machine-tuned",
                                      created_at=datetime.datetime.now(datetime.timezone.utc)
                                      .strftime("%Y-%m-%dT%H:%M:%SZ"),
                                      host=host or platform.node())
    return best_p


# ---------------------------------------------------------------------------
# The reference's tuning procedure (src/tuner.py:96-333) on B200 timings:
# timing grid -> labels with margin ratios -> near-tie filter -> two
# maximum-margin lines over (r, n) (svm.py) -> p4 / p8 -> TuningParams.
# Same names and contracts as the reference's ``permanent.tuner``.
# ---------------------------------------------------------------------------
import statistics  # noqa: E402
import time  # noqa: E402
from dataclasses import dataclass, field  # noqa: E402

import numpy as np  # noqa: E402

from . import svm  # noqa: E402
from .core import ElementKind  # noqa: E402

GRID_N = range(2, 25)                     # the reference's grid (tuner.py:27)
B200_GRID_N = range(2, 35)                # the B200 fit: walks are cheap up to n = 34
GRID_RATIOS = (1 / 8, 1 / 4, 3 / 8, 1 / 2, 5 / 8, 3 / 4, 7 / 8, 1.0)
COMBINATORIC_MAX_COLS = 14                # CPU budgets of algorithm_feasible (tuner.py:32-36)
COMBINATORIC_MAX_STEPS = 50_000_000
WALK_MAX_COLS = 26
NEAR_TIE_FILTER = 1.05
MIN_SAMPLE_SECONDS = 200e-6


@dataclass(frozen=True)
class BenchmarkSample:
    """Median time of one algorithm at one grid shape (tuner.py:44-55)."""

    algorithm: object
    m: int
    n: int
    ratio: float
    median_time: float
    trials: int
    kind: ElementKind = ElementKind.FLOAT64
    feasible: bool = True


@dataclass(frozen=True)
class LabeledPoint:
    """A grid cell labeled with its fastest algorithm; ``margin_ratio`` =
    runner-up / winner (inf with one feasible algorithm)."""

    r: float
    n: int
    m: int
    label: object
    margin_ratio: float
    best_median: float = 0.0


@dataclass(frozen=True)
class SeparatingPlane:
    """weight_r r + weight_n n + bias = 0; the first trained class is on the
    positive side; ``fallback`` when the classes were not separable."""

    weight_r: float
    weight_n: float
    bias: float
    fallback: bool = False

    def evaluate(self, r, n):
        return self.weight_r * r + self.weight_n * n + self.bias


@dataclass(frozen=True)
class TuningReport:
    params: TuningParams
    grid: list
    plane_small: SeparatingPlane
    plane_large: SeparatingPlane
    intersection: object = None
    timings: dict = field(default_factory=dict)


def algorithm_feasible(alg, m: int, n: int, comb_steps: int = COMBINATORIC_MAX_STEPS,
                       comb_cols: int = COMBINATORIC_MAX_COLS, walk_cols: int = WALK_MAX_COLS) -> bool:
    """Whether a cell is affordable on the tuning grid.  Defaults are the
    reference's CPU budgets (tuner.py:96-102); the B200 grid passes its own
    (``B200_BUDGET``)."""
    from .algorithms import AlgorithmId

    if alg is AlgorithmId.COMBINATORIC:
        return n <= comb_cols and m * math.perm(n, m) <= comb_steps
    return n <= walk_cols


# the B200 grid: the GPU combinatoric kernel handles ~1e9 row-steps in tens
# of ms, and the walks reach n = 34 in ~30 ms
B200_BUDGET = dict(comb_steps=2_000_000_000, comb_cols=20, walk_cols=34)


def time_algorithm(alg, m, n, trials=5, seed=None, budget=None) -> BenchmarkSample:
    """Median wall time of ``run_algorithm`` (the public mid-level call: host
    matrix in, Python value out, kernels in between) on fresh U[-1,1]
    float64 matrices, repeats amortized to >= MIN_SAMPLE_SECONDS
    (tuner.py:108-135)."""
    from .algorithms import run_algorithm
    from .core import as_matrix

    if trials < 3:
        raise ValueError(f"need at least 3 trials, got {trials}")
    if not algorithm_feasible(alg, m, n, **(budget or {})):
        return BenchmarkSample(alg, m, n, m / n, math.inf, 0, feasible=False)
    g = np.random.default_rng(seed)
    mats = [as_matrix(g.uniform(-1.0, 1.0, (m, n))) for _ in range(trials + 1)]
    t0 = time.perf_counter()
    run_algorithm(mats[0], alg)
    warm = time.perf_counter() - t0
    reps = max(1, min(200, round(MIN_SAMPLE_SECONDS / max(warm, 1e-9))))
    ts = []
    for mat in mats[1:]:
        t0 = time.perf_counter()
        for _ in range(reps):
            run_algorithm(mat, alg)
        ts.append((time.perf_counter() - t0) / reps)
    return BenchmarkSample(alg, m, n, m / n, statistics.median(ts), trials)


def grid_shapes(n_range=GRID_N, ratios=GRID_RATIOS):
    """Deduplicated (m, n) cells, m = max(1, round(r n)) (tuner.py:138-149)."""
    seen, out = set(), []
    for n in n_range:
        for r in ratios:
            m = max(1, round(r * n))
            if m <= n and (m, n) not in seen:
                seen.add((m, n))
                out.append((m, n))
    return out


def measure_grid(n_range=GRID_N, ratios=GRID_RATIOS, trials=5, seed=0, budget=None) -> dict:
    """{(m, n): {alg: median seconds}} over the feasible algorithms."""
    from .algorithms import AlgorithmId

    timings, s = {}, seed
    for m, n in grid_shapes(n_range, ratios):
        cell = {}
        for alg in AlgorithmId:
            s += 1
            smp = time_algorithm(alg, m, n, trials=trials, seed=s, budget=budget)
            if smp.feasible:
                cell[alg.value] = smp.median_time
        timings[(m, n)] = cell
    return timings


def label_grid(timings: dict) -> list:
    """Label each cell by its fastest algorithm, in grid order; cells with no
    feasible algorithm are omitted."""
    from .algorithms import AlgorithmId

    pts = []
    for (m, n), t in timings.items():
        feas = sorted((v, a) for a, v in t.items() if math.isfinite(v))
        if not feas:
            continue
        margin = feas[1][0] / feas[0][0] if len(feas) > 1 else math.inf
        pts.append(LabeledPoint(m / n, n, m, AlgorithmId(feas[0][1]), margin, feas[0][0]))
    return pts


def build_label_grid(n_range=GRID_N, ratios=GRID_RATIOS, trials=5, seed=0, budget=None) -> list:
    """Time every algorithm on every cell and label the winners (tuner.py:152-173)."""
    return label_grid(measure_grid(n_range, ratios, trials, seed, budget))


def detect_small_square_cutoff(grid) -> int:
    """Largest n with combinatoric fastest on every square up to n (else 1)."""
    from .algorithms import AlgorithmId

    cut = 1
    for p in sorted((p for p in grid if p.m == p.n and p.n >= 2), key=lambda p: p.n):
        if p.label is not AlgorithmId.COMBINATORIC:
            break
        cut = p.n
    return cut


def fit_hard_margin_svm(points, class_a, class_b, near_tie: float = NEAR_TIE_FILTER) -> SeparatingPlane:
    """Maximum-margin line between two labels over (r, n) after dropping
    near-ties; ``class_a`` on the positive side.  Not separable: the
    weighted minimum-cost line (misrouting costs margin_ratio - 1, capped at
    9), flagged ``fallback`` (tuner.py:187-213)."""
    kept = [p for p in points if p.label in (class_a, class_b) and p.margin_ratio >= near_tie]
    for cls in (class_a, class_b):
        if not any(p.label is cls for p in kept):
            raise ValueError(f"no retained training points labeled {cls.value}")
    X = np.array([[p.r, p.n] for p in kept], dtype=float)
    y = np.array([1.0 if p.label is class_a else -1.0 for p in kept])
    fit = svm.max_margin_plane(X, y)
    if fit is not None:
        w, b, _ = fit
        return SeparatingPlane(float(w[0]), float(w[1]), float(b))
    wts = np.array([min(p.margin_ratio, 10.0) - 1.0 for p in kept])
    w, b, _ = svm.min_misclassification_plane(X, y, weights=wts)
    return SeparatingPlane(float(w[0]), float(w[1]), float(b), fallback=True)


def plane_intersection(p: SeparatingPlane, q: SeparatingPlane):
    """(r, n) where the two lines cross (Cramer's rule), or None when they
    are parallel to within 1e-12 of the coefficient scale."""
    det = p.weight_r * q.weight_n - p.weight_n * q.weight_r
    scale = max(1.0, abs(p.weight_r), abs(p.weight_n), abs(q.weight_r), abs(q.weight_n)) ** 2
    if abs(det) < 1e-12 * scale:
        return None
    r = (-p.bias * q.weight_n + q.bias * p.weight_n) / det
    n = (-q.bias * p.weight_r + p.bias * q.weight_r) / det
    return float(r), float(n)


def assemble_params(grid, plane1: SeparatingPlane, plane2: SeparatingPlane, p4, p8) -> TuningParams:
    """p1..p3 from plane1 (combinatoric positive), p5..p7 from plane2 (Glynn
    positive), p4 clamped to p8; a plane on which every relevant training
    point lies is rejected as orientation-ambiguous (tuner.py:226-250)."""
    from .algorithms import AlgorithmId

    C, G, R = AlgorithmId.COMBINATORIC, AlgorithmId.GLYNN, AlgorithmId.RYSER
    for plane, pos, neg in ((plane1, C, G), (plane2, G, R)):
        rel = [p for p in grid if p.label in (pos, neg)]
        if rel and all(abs(plane.evaluate(p.r, p.n)) <= 1e-12 for p in rel):
            raise ValueError("separating plane orientation is ambiguous: every training point lies on the plane")
    stamp = datetime.datetime.now(datetime.timezone.utc).isoformat(timespec="seconds")
    return TuningParams(p1=plane1.weight_r, p2=plane1.weight_n, p3=plane1.bias, p4=float(min(p4, p8)),
                        p5=plane2.weight_r, p6=plane2.weight_n, p7=plane2.bias, p8=float(p8),
                        source="machine-tuned", created_at=stamp,
                        host=f"{platform.node()} ({platform.machine()})")


def _fit_or_default(points, class_a, class_b) -> SeparatingPlane:
    """fit_hard_margin_svm, or a constant-sign line steering every cell away
    from a class that never wins decisively (tuner.py:253-266)."""
    won = {p.label for p in points if p.margin_ratio >= NEAR_TIE_FILTER}
    if class_a in won and class_b in won:
        return fit_hard_margin_svm(points, class_a, class_b)
    return SeparatingPlane(0.0, -1.0, 0.0) if class_a not in won else SeparatingPlane(0.0, 1.0, 0.0)


def _derive_p8(plane1, plane2, grid, max_n):
    """Regime boundary: the lines' crossing column, else one past the last
    combinatoric win; raised to cover every decisive (>= 1.25x)
    combinatoric cell, clamped to [2, max_n] (tuner.py:269-283)."""
    from .algorithms import AlgorithmId

    inter = plane_intersection(plane1, plane2)
    comb = [p for p in grid if p.label is AlgorithmId.COMBINATORIC]
    if inter is not None and 2 <= inter[1] <= max_n:
        p8 = round(inter[1])
    else:
        p8 = max(p.n for p in comb) + 1 if comb else 2
    decisive = [p.n for p in comb if p.margin_ratio >= 1.25]
    if decisive:
        p8 = max(p8, max(decisive))
    return max(2, min(p8, max_n)), inter


def _total_slowdown(params, timings):
    from .dispatch import select_algorithm

    tot = 0.0
    for (m, n), t in timings.items():
        pick = select_algorithm(m, n, params).value
        tot += (t[pick] / min(t.values())) if pick in t else 1e6
    return tot


def run_tuning(n_range=GRID_N, ratios=GRID_RATIOS, trials=5, seed=0, timings=None, budget=None) -> TuningReport:
    """The reference's pipeline (tuner.py:286-310): label grid, p4 from the
    square cutoff, the combinatoric/Glynn line on the unpinned cells, the
    Glynn/Ryser line fit twice (second pass on the large regime the first
    located), p8 from their crossing.  ``timings`` ({(m, n): {alg: s}})
    skips the measurement and fits recorded B200 timings."""
    from .algorithms import AlgorithmId

    C, G, R = AlgorithmId.COMBINATORIC, AlgorithmId.GLYNN, AlgorithmId.RYSER
    if timings is None:
        timings = measure_grid(n_range, ratios, trials, seed, budget)
    grid = label_grid(timings)
    max_n = max(p.n for p in grid)
    p4 = detect_small_square_cutoff(grid)
    unpinned = [p for p in grid if not (p.m == p.n and p.n <= p4)]
    plane1 = _fit_or_default(unpinned, C, G)
    plane2 = _fit_or_default(grid, G, R)
    p8, _ = _derive_p8(plane1, plane2, grid, max_n)
    large = [p for p in grid if p.n > p8]
    plane2 = _fit_or_default(large or grid, G, R)
    p8, inter = _derive_p8(plane1, plane2, grid, max_n)
    params = assemble_params(grid, plane1, plane2, p4, p8)
    return TuningReport(params, grid, plane1, plane2, inter, timings)


def evaluate_dispatch(params: TuningParams, shapes, trials: int = 5, seed: int = 0, budget=None):
    """(m, n, chosen, slowdown) per probe shape: the selected algorithm's
    median time over the fastest feasible one's, timed on the GPU engine
    (the acceptance probe of tuner.py:313-333)."""
    from .algorithms import AlgorithmId
    from .dispatch import select_algorithm

    out, s = [], seed + 90000
    for m, n in shapes:
        chosen = select_algorithm(m, n, params)
        med = {}
        for alg in AlgorithmId:
            s += 1
            smp = time_algorithm(alg, m, n, trials=trials, seed=s, budget=budget)
            if smp.feasible:
                med[alg] = smp.median_time
        out.append((m, n, chosen, med[chosen] / min(med.values()) if chosen in med else math.inf))
    return out
