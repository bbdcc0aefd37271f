"""Tuning file v1 (line-oriented key=value) and the B200 crossover tuner.

File format: the reference's (/root/reference/pkg/src/permanent/tuner.py:340-383):
``format_version=1``, ``source``, ``host``, ``created_at`` and ``p1``..``p8``,
one key per line, floats in shortest round-trip form; unknown, duplicate or
missing keys and other versions are rejected with ValueError.

The tuner reuses the reference's *procedure* (tuner.py:286-310: time every
algorithm over an (m, n) grid, label each cell with its fastest algorithm,
fit the two separating lines and the regime boundary p8) with B200 kernel
timings in place of CPU timings; the lines are fitted by exhaustive search
over a parameter grid (minimum total slowdown), a robust stand-in for the
reference's hard-margin SVM (src/svm.py) when labels are not separable.
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
            if c1 + c2 < best_c:
                best_c = c1 + c2
                best_p = TuningParams(p1=b1[0], p2=b1[1], p3=b1[2], p4=float(p4), p5=b2[0], p6=b2[1],
                                      p7=b2[2], p8=float(p8), source="machine-tuned",
                                      created_at=datetime.datetime.now(datetime.timezone.utc)
                                      .strftime("%Y-%m-%dT%H:%M:%SZ"),
                                      host=host or platform.node())
    return best_p
