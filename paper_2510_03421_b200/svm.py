"""Linear separators in the (r, n) plane for the dispatch tuner.

Same contracts as the reference's ``permanent.svm``
(/root/reference/pkg/src/permanent/svm.py:56-129), computed differently:

* ``max_margin_plane(X, y)`` -- the hard-margin SVM.  Two finite point sets
  are strictly linearly separable iff their convex hulls are disjoint, and
  then the widest separating strip is bounded by the perpendicular bisector
  of the closest pair of hull points (p in hull(+), q in hull(-)); its full
  width is |p - q|.  Hulls by Andrew's monotone chain; the closest pair is a
  vertex pair or a vertex against the interior of an edge.  Returns
  ``(w, b, gap)`` scaled so that min_i y_i (w . x_i + b) = 1, or None when
  the classes overlap (or one is empty).
* ``min_misclassification_plane(X, y, angles, weights)`` -- the fallback for
  inseparable labels: over ``angles`` directions u and every threshold
  between consecutive projections, minimize the weight of misrouted points
  (points strictly above the threshold are called +1); ties go to fewer
  misrouted points, then to the wider gap around the threshold.  Returns
  ``(w, b, cost)``.  All directions are evaluated in one vectorized pass.
"""
from __future__ import annotations

import numpy as np


def _cross(o, a, b) -> float:
    return (a[0] - o[0]) * (b[1] - o[1]) - (a[1] - o[1]) * (b[0] - o[0])


def _hull(P: np.ndarray) -> list:
    """Convex hull vertices (counter-clockwise, no collinear interior
    points); one point or a segment's two endpoints for degenerate sets."""
    pts = sorted({(float(x), float(y)) for x, y in P})
    if len(pts) <= 2:
        return [np.array(p) for p in pts]
    lower, upper = [], []
    for p in pts:
        while len(lower) >= 2 and _cross(lower[-2], lower[-1], p) <= 0:
            lower.pop()
        lower.append(p)
    for p in reversed(pts):
        while len(upper) >= 2 and _cross(upper[-2], upper[-1], p) <= 0:
            upper.pop()
        upper.append(p)
    return [np.array(p) for p in lower[:-1] + upper[:-1]]


def _edges(h: list):
    if len(h) == 2:
        return [(h[0], h[1])]
    if len(h) < 2:
        return []
    return [(h[i], h[(i + 1) % len(h)]) for i in range(len(h))]


def _closest_pair(ha: list, hb: list):
    """Closest (p, q), p on hull a, q on hull b (boundaries)."""
    best = None

    def consider(p, q):
        nonlocal best
        d = float((p - q) @ (p - q))
        if best is None or d < best[0]:
            best = (d, p, q)

    for p in ha:
        for q in hb:
            consider(p, q)
    for verts, edges, flip in ((ha, _edges(hb), False), (hb, _edges(ha), True)):
        for v in verts:
            for s, e in edges:
                u = e - s
                uu = float(u @ u)
                if uu <= 0.0:
                    continue
                t = float((v - s) @ u) / uu
                if 0.0 < t < 1.0:
                    foot = s + t * u
                    consider(foot, v) if flip else consider(v, foot)
    return best[1], best[2]


def max_margin_plane(X: np.ndarray, y: np.ndarray):
    """Widest-margin line w . x + b = 0 with the y = +1 points on its
    positive side; ``(w, b, gap)`` with min_i y_i (w . x_i + b) = 1 and gap =
    2 / |w| the strip width, or None if the classes are not strictly
    separable."""
    X = np.asarray(X, dtype=float)
    y = np.asarray(y, dtype=float)
    pos, neg = X[y > 0], X[y <= 0]
    if len(pos) == 0 or len(neg) == 0:
        return None
    p, q = _closest_pair(_hull(pos), _hull(neg))
    u = p - q
    if float(u @ u) <= 1e-30:
        return None
    w0 = u
    b0 = -float(u @ (p + q)) / 2.0
    scores = y * (X @ w0 + b0)
    smin = float(scores.min())
    if smin <= 0.0:  # hulls overlap: one contains the other's boundary pair
        return None
    w = w0 / smin
    return w, b0 / smin, 2.0 / float(np.linalg.norm(w))


def min_misclassification_plane(X: np.ndarray, y: np.ndarray, angles: int = 3600, weights=None):
    """Minimum misrouted weight over a direction x threshold sweep (see the
    module doc); ``(w, b, cost)`` with w a unit vector."""
    X = np.asarray(X, dtype=float)
    y = np.asarray(y, dtype=float)
    npts = len(y)
    wts = np.ones(npts) if weights is None else np.asarray(weights, dtype=float)
    th = 2.0 * np.pi * np.arange(angles) / angles
    U = np.stack([np.cos(th), np.sin(th)], axis=1)          # [angles, 2]
    proj = U @ X.T                                           # [angles, npts]
    order = np.argsort(proj, axis=1, kind="stable")
    ps = np.take_along_axis(proj, order, axis=1)
    isp = (y[order] > 0)
    isn = (y[order] < 0)
    wt = wts[order]
    zero = np.zeros((angles, 1))
    # cut i (0..npts): the i lowest projections are called -1, the rest +1
    pos_below = np.concatenate([zero, np.cumsum(wt * isp, axis=1)], axis=1)
    neg_above = np.concatenate([np.cumsum((wt * isn)[:, ::-1], axis=1)[:, ::-1], zero], axis=1)
    cost = pos_below + neg_above
    errs = (np.concatenate([zero, np.cumsum(isp, axis=1)], axis=1)
            + np.concatenate([np.cumsum(isn[:, ::-1], axis=1)[:, ::-1], zero], axis=1))
    gap = np.zeros((angles, npts + 1))
    if npts > 1:
        gap[:, 1:npts] = ps[:, 1:] - ps[:, :-1]
    # lexicographic (cost, errors, -gap), first direction / lowest cut on ties
    flat = np.lexsort(((-gap).ravel(), errs.ravel(), cost.ravel()))[0]
    a, i = divmod(int(flat), npts + 1)
    if i == 0:
        thr = ps[a, 0] - 1.0
    elif i == npts:
        thr = ps[a, -1] + 1.0
    else:
        thr = 0.5 * (ps[a, i - 1] + ps[a, i])
    return U[a].copy(), -float(thr), float(cost[a, i])
