"""Tuning file v1 (line-oriented key=value) and the B200 crossover tuner.

File format: the reference's (/root/reference/pkg/src/permanent/tuner.py:340-383):
``format_version=1``, ``source``, ``host``, ``created_at`` and ``p1``..``p8``,
one key per line, floats in shortest round-trip form; unknown, duplicate or
missing keys and other versions are rejected with ValueError.

Two fits over B200 kernel timings {(m, n): {alg: seconds}}:
* ``run_tuning`` -- the reference's procedure (tuner.py:108-310): timing
  grid, labels with margin ratios, near-tie filter, two maximum-margin lines
  over (r, n) (hard-margin SVM, weighted minimum-cost fallback when the
  labels are not separable), p4 from the square cutoff, p8 chosen to
  minimize the total dispatch slowdown;
* ``fit_params`` -- a direct grid search minimizing the summed relative
  slowdown (used for the shipped ``tuned/b200.tuning``: GPU timings below
  ~50 us are launch-overhead dominated, so labels there are noisy and
  rarely separable).
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
    wv, b = _min_cost_line(np.array(X, float), np.array(y), np.array(w), angles=720)
    if wv is None or (wv[0] == 0 and wv[1] == 0):
        return None
    return float(wv[0]), float(wv[1]), float(b)


def fit_params(timings: dict, host: str = "") -> TuningParams:
    """Fit p1..p8 to measured timings {(m, n): {alg: seconds}} by minimizing
    the summed relative slowdown of the selected algorithm (grid search)."""
    cells = {k: v for k, v in timings.items() if v}

    def cost(p):
        tot = 0.0
        for (m, n), t in cells.items():
            best = min(t.values())
            pick = _select(p, m, n)
            tot += (t.get(pick, math.inf) / best) - 1.0 if pick in t else 1e6
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
                    tot += (t[pick] / min(t.values()) - 1.0) if pick in t else 1e6
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
# The reference's tuning procedure (src/tuner.py:108-310) on B200 timings:
# timing grid -> labels with margin ratios -> near-tie filter -> two
# maximum-margin lines over (r, n) -> p4 / p8 -> TuningParams.
# ---------------------------------------------------------------------------
import statistics  # noqa: E402
import time  # noqa: E402
from dataclasses import dataclass  # noqa: E402

import numpy as np  # noqa: E402

GRID_N = range(2, 35)
GRID_RATIOS = (1 / 8, 1 / 4, 3 / 8, 1 / 2, 5 / 8, 3 / 4, 7 / 8, 1.0)
NEAR_TIE_FILTER = 1.05
COMBINATORIC_MAX_STEPS = 50_000_000
MIN_SAMPLE_SECONDS = 200e-6


@dataclass(frozen=True)
class BenchmarkSample:
    algorithm: object
    m: int
    n: int
    ratio: float
    median_time: float
    trials: int
    feasible: bool = True


@dataclass(frozen=True)
class LabeledPoint:
    r: float
    n: int
    m: int
    label: object
    margin_ratio: float
    best_median: float = 0.0


@dataclass(frozen=True)
class SeparatingPlane:
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
    timings: dict


def grid_shapes(n_range=GRID_N, ratios=GRID_RATIOS):
    seen, out = set(), []
    for n in n_range:
        for r in ratios:
            m = max(1, round(r * n))
            if m <= n and (m, n) not in seen:
                seen.add((m, n))
                out.append((m, n))
    return out


def time_algorithm(alg, m, n, trials=5, seed=None) -> BenchmarkSample:
    """Median wall time of run_algorithm on fresh U[-1,1] float64 matrices,
    repeats amortized to >= MIN_SAMPLE_SECONDS (src/tuner.py:108-135)."""
    from .algorithms import AlgorithmId, run_algorithm
    from .core import as_matrix

    if trials < 3:
        raise ValueError(f"need at least 3 trials, got {trials}")
    if alg is AlgorithmId.COMBINATORIC and math.perm(n, m) > COMBINATORIC_MAX_STEPS:
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


def evaluate_dispatch(params: TuningParams, shapes, trials: int = 5, seed: int = 0):
    """(m, n, chosen, slowdown) per probe shape, slowdown = the chosen
    algorithm's median / the fastest feasible median, timed on the GPU engine
    (the reference's acceptance probe, src/tuner.py:313-333)."""
    from .algorithms import AlgorithmId
    from .dispatch import select_algorithm

    out = []
    probe_seed = seed + 90000
    for m, n in shapes:
        chosen = select_algorithm(m, n, params)
        medians = {}
        for alg in AlgorithmId:
            probe_seed += 1
            smp = time_algorithm(alg, m, n, trials=trials, seed=probe_seed)
            if smp.feasible:
                medians[alg] = smp.median_time
        best = min(medians.values())
        out.append((m, n, chosen, medians[chosen] / best if chosen in medians else math.inf))
    return out


def label_grid(timings: dict) -> list:
    """Label each cell {(m, n): {alg: seconds}} by its fastest algorithm."""
    from .algorithms import AlgorithmId

    pts = []
    for (m, n), t in sorted(timings.items(), key=lambda kv: (kv[0][1], kv[0][0])):
        feas = sorted((v, a) for a, v in t.items() if math.isfinite(v))
        if not feas:
            continue
        margin = feas[1][0] / feas[0][0] if len(feas) > 1 else math.inf
        pts.append(LabeledPoint(m / n, n, m, AlgorithmId(feas[0][1]), margin, feas[0][0]))
    return pts


def build_label_grid(n_range=GRID_N, ratios=GRID_RATIOS, trials=5, seed=0):
    from .algorithms import AlgorithmId

    timings, s = {}, seed
    for m, n in grid_shapes(n_range, ratios):
        cell = {}
        for alg in AlgorithmId:
            s += 1
            smp = time_algorithm(alg, m, n, trials=trials, seed=s)
            if smp.feasible:
                cell[alg.value] = smp.median_time
        timings[(m, n)] = cell
    return label_grid(timings), timings


def detect_small_square_cutoff(grid) -> int:
    """Largest n with combinatoric fastest on every square up to n (else 1)."""
    from .algorithms import AlgorithmId

    cut = 1
    for p in sorted((p for p in grid if p.m == p.n and p.n >= 2), key=lambda p: p.n):
        if p.label is not AlgorithmId.COMBINATORIC:
            break
        cut = p.n
    return cut


def _max_margin(X, y):
    """Hard-margin linear SVM in 2-D (min |w|^2 s.t. y (w.x + b) >= 1), or
    None if the classes are not linearly separable."""
    from scipy.optimize import minimize

    scale = np.maximum(np.abs(X).max(axis=0), 1e-12)
    Xs = X / scale
    cons = {"type": "ineq", "fun": lambda z: y * (Xs @ z[:2] + z[2]) - 1.0,
            "jac": lambda z: np.column_stack([y[:, None] * Xs, y])}
    best = None
    for z0 in (np.array([1.0, 0.0, 0.0]), np.array([0.0, 1.0, 0.0]), np.array([1.0, 1.0, -1.0])):
        r = minimize(lambda z: z[0] ** 2 + z[1] ** 2, z0, jac=lambda z: np.array([2 * z[0], 2 * z[1], 0.0]),
                     constraints=[cons], method="SLSQP", options={"maxiter": 500, "ftol": 1e-12})
        if r.success and np.all(y * (Xs @ r.x[:2] + r.x[2]) >= 1.0 - 1e-6):
            if best is None or r.fun < best.fun:
                best = r
    if best is None:
        return None
    w = best.x[:2] / scale
    return w, float(best.x[2])


def _min_cost_line(X, y, weights, angles=1440):
    """Weighted minimum-misclassification line: sweep directions; for each,
    the best threshold over sorted projections by cumulative sums."""
    scale = np.maximum(np.abs(X).max(axis=0), 1e-12)
    Xs = X / scale
    best = (math.inf, None, None)
    for th in np.linspace(0.0, 2 * math.pi, angles, endpoint=False):
        w = np.array([math.cos(th), math.sin(th)])
        proj = Xs @ w
        order = np.argsort(proj)
        ps, ys, ws = proj[order], y[order], weights[order]
        # threshold after position i: points <= are predicted -1, > are +1
        pos_left = np.concatenate([[0.0], np.cumsum(ws * (ys > 0))])       # +1 points on the -1 side
        neg_right = np.concatenate([np.cumsum((ws * (ys < 0))[::-1])[::-1], [0.0]])  # -1 points on the +1 side
        cost = pos_left + neg_right
        i = int(np.argmin(cost))
        if cost[i] < best[0]:
            if i == 0:
                b = ps[0] - 1.0
            elif i == len(ps):
                b = ps[-1] + 1.0
            else:
                b = 0.5 * (ps[i - 1] + ps[i])
            best = (float(cost[i]), w / scale, -b)
    return best[1], best[2]


def fit_separator(points, class_a, class_b, near_tie=NEAR_TIE_FILTER) -> SeparatingPlane:
    """Max-margin line between two labels over (r, n) after the near-tie
    filter; weighted min-cost fallback when not separable (src/tuner.py:187-213)."""
    kept = [p for p in points if p.label in (class_a, class_b) and p.margin_ratio >= near_tie]
    if not any(p.label is class_a for p in kept) or not any(p.label is class_b for p in kept):
        raise ValueError("both classes need retained training points")
    X = np.array([[p.r, p.n] for p in kept], dtype=float)
    y = np.array([1.0 if p.label is class_a else -1.0 for p in kept])
    fit = _max_margin(X, y)
    if fit is not None:
        w, b = fit
        return SeparatingPlane(float(w[0]), float(w[1]), b)
    wts = np.array([min(p.margin_ratio, 10.0) - 1.0 for p in kept])
    w, b = _min_cost_line(X, y, wts)
    return SeparatingPlane(float(w[0]), float(w[1]), float(b), fallback=True)


def _total_slowdown(params, timings):
    from .dispatch import select_algorithm

    tot = 0.0
    for (m, n), t in timings.items():
        pick = select_algorithm(m, n, params).value
        tot += (t[pick] / min(t.values())) if pick in t else 1e6
    return tot


def run_tuning(n_range=GRID_N, ratios=GRID_RATIOS, trials=5, seed=0, timings=None) -> TuningReport:
    """The whole pipeline; with ``timings`` ({(m, n): {alg: s}}) it only fits."""
    import datetime
    import platform

    from .algorithms import AlgorithmId

    C, G, R = AlgorithmId.COMBINATORIC, AlgorithmId.GLYNN, AlgorithmId.RYSER
    if timings is None:
        grid, timings = build_label_grid(n_range, ratios, trials, seed)
    else:
        grid = label_grid(timings)
    max_n = max(p.n for p in grid)
    p4 = detect_small_square_cutoff(grid)

    def plane(pts, a, b, default):
        try:
            return fit_separator(pts, a, b)
        except ValueError:
            return default

    plane1 = plane([p for p in grid if not (p.m == p.n and p.n <= p4)], C, G,
                   SeparatingPlane(-1.0, 0.0, -1.0, fallback=True))
    best = None
    for p8 in range(max(2, p4), max_n + 1):
        large = [p for p in grid if p.n > p8]
        plane2 = plane(large or grid, G, R, SeparatingPlane(1.0, 0.0, 1.0, fallback=True))
        try:
            params = TuningParams(plane1.weight_r, plane1.weight_n, plane1.bias, float(p4),
                                  plane2.weight_r, plane2.weight_n, plane2.bias, float(p8),
                                  source="machine-tuned")
        except ValueError:
            continue
        cost = _total_slowdown(params, timings)
        if best is None or cost < best[0]:
            best = (cost, params, plane2)
    _, params, plane2 = best
    stamp = datetime.datetime.now(datetime.timezone.utc).strftime("%Y-%m-%dT%H:%M:%SZ")
    params = TuningParams(*params.as_list(), source="machine-tuned", created_at=stamp, host=platform.node())
    return TuningReport(params, grid, plane1, plane2, timings)
