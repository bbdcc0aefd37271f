"""The zero-copy single-permanent path (round 2, DESIGN 2.3b) against the
CPU oracle, over every branch it has:

- the chunked walk kernel with the setup as kernel parameters (real P <= 26,
  complex P <= 18, weighted rectangular Ryser with m <= 10 / complex m <= 5)
  and the result through a mapped flag;
- the one-warp kernel below 256 Gray steps (Glynn n <= 8, Ryser n <= 7);
- the staged path past the inline size, and a caller's stream (stream-ordered
  copies, the batch-of-one kernels for tiny walks), which must agree with the
  default-stream result to within rounding;
- the magnitude sum through the zero-copy path, pinned to the oracle's.

Tolerance: metric (ii) 1e-10 with the oracle's magnitude sum (north_star)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import paper_2510_03421_b200 as P
from conftest import scaled_err
from oracle import oracle as O
from paper_2510_03421_b200 import _lib

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _oracle(alg, a):
    return O.dd_permanent(alg, a, nthreads=8) if a.shape[1] >= 16 else O.permanent(alg, a)[0]


def _call(alg, a, stream=None):
    """perm_{glynn,ryser}_{f64,c128} on a host matrix; stream None = the
    default-stream (zero-copy) route."""
    lib = _lib.load()
    cplx = np.iscomplexobj(a)
    a = np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)
    m, n = a.shape
    out = _lib.out_buf(2)
    mg = C.c_double(0.0)
    fn = getattr(lib, f"perm_{alg}_{'c128' if cplx else 'f64'}")
    st = fn(m, n, C.c_void_p(a.ctypes.data), n, 0, out, C.byref(mg), C.c_void_p(stream) if stream else None)
    _lib.check(st, f"{alg} {m}x{n}")
    return (complex(out[0], out[1]) if cplx else float(out[0])), mg.value


def _mat(rng, m, n, cplx):
    a = rng.uniform(-1, 1, (m, n)) / np.sqrt(n)
    if cplx:
        a = a + 1j * rng.uniform(-1, 1, (m, n)) / np.sqrt(n)
    return a


@pytest.mark.parametrize("cplx", [False, True])
def test_square_walks_all_sizes(rng, cplx):
    """Glynn and Ryser n = 1..24 (real) / 1..20 (complex): the one-warp
    kernel, the inline chunked kernel and (complex n > 18) the staged one."""
    top = 20 if cplx else 24
    for n in range(1, top + 1):
        a = _mat(rng, n, n, cplx)
        M = O.glynn_magnitude_sum(a)
        for alg in ("glynn", "ryser"):
            v = (P.glynn if alg == "glynn" else P.ryser)(a)
            ref = _oracle(alg, a)
            assert scaled_err(v, ref, M) <= TOL, (alg, n, v, ref)


@pytest.mark.parametrize("cplx", [False, True])
def test_rectangular_walks(rng, cplx):
    """Rectangular Glynn (ones-padded, pre-scaled) and rectangular Ryser
    (weighted walk with inline weights, or the combination order): shapes on
    both sides of the cost model's crossover and of the inline limits."""
    shapes = [(1, 3), (2, 5), (3, 7), (2, 9), (4, 9), (3, 12), (5, 14), (6, 16), (8, 18), (10, 20), (3, 21),
              (12, 22)]
    for m, n in shapes:
        a = _mat(rng, m, n, cplx)
        M = O.glynn_magnitude_sum(a)
        ref = O.permanent("combinatoric", a)[0] if m <= 6 else _oracle("ryser", a)
        for fn in (P.glynn, P.ryser, P.ryser_rectangular, P.opt):
            v = fn(a)
            assert scaled_err(v, ref, M) <= TOL, (fn.__name__, m, n, v, ref)


def test_caller_stream_matches_default_stream(rng):
    """A caller's stream takes the staged / batch-of-one routes: same value
    (up to summation order) and the same magnitude sum as the zero-copy one."""
    torch = pytest.importorskip("torch")
    s = torch.cuda.Stream()
    for cplx in (False, True):
        for m, n in ((4, 4), (7, 7), (8, 8), (12, 12), (16, 16), (20, 20), (3, 9), (5, 13)):
            a = _mat(rng, m, n, cplx)
            M = O.glynn_magnitude_sum(a)
            for alg in ("glynn", "ryser"):
                v0, m0 = _call(alg, a)
                v1, m1 = _call(alg, a, stream=s.cuda_stream)
                s.synchronize()
                assert scaled_err(v0, v1, M) <= 1e-13, (alg, m, n, cplx)
                if m == n or alg == "glynn":
                    assert abs(m0 - m1) <= 1e-12 * max(m0, m1), (alg, m, n)


def test_zero_copy_magsum_pinned_to_oracle(rng):
    """The magnitude sum returned through the mapped result slot equals the
    oracle's Glynn magnitude sum (square and ones-padded rectangles)."""
    for m, n in ((5, 5), (9, 9), (16, 16), (22, 22), (4, 10), (11, 17)):
        a = _mat(rng, m, n, False)
        _, mg = _call("glynn", a)
        ref = O.glynn_magnitude_sum(a)
        assert abs(mg - ref) <= 1e-12 * ref, (m, n, mg, ref)


def test_back_to_back_calls_do_not_mix_results(rng):
    """Consecutive zero-copy calls of different sizes and kinds (the mapped
    slot and its sequence flag are reused): each returns its own value."""
    mats = [_mat(rng, n, n, c) for n, c in ((6, False), (20, False), (9, True), (24, False), (3, False),
                                             (14, True), (17, False))]
    refs = [_oracle("glynn", a) for a in mats]
    Ms = [O.glynn_magnitude_sum(a) for a in mats]
    for _ in range(3):
        for a, r, M in zip(mats, refs, Ms):
            assert scaled_err(P.glynn(a), r, M) <= TOL


def test_repeat_ms_entry_point(rng):
    """perm_walk_repeat_ms: a positive per-launch device time, errors on bad
    arguments."""
    lib = _lib.load()
    a = np.ascontiguousarray(_mat(rng, 20, 20, False))
    ms = _lib.out_buf(1)
    _lib.check(lib.perm_walk_repeat_ms(_lib.ALG_GLYNN, 0, 20, 20, C.c_void_p(a.ctypes.data), 20, 20, ms), "repeat")
    assert 0.0 < ms[0] < 5.0
    assert lib.perm_walk_repeat_ms(_lib.ALG_COMBINATORIC, 0, 20, 20, C.c_void_p(a.ctypes.data), 20, 20, ms) != 0


def _same_special(x, ref):
    """NaN where the reference has NaN, the same infinities, the same signed
    zeros, finite values within 1e-12 relative."""
    import math

    if math.isnan(ref):
        return math.isnan(x)
    if math.isinf(ref) or ref == 0.0:
        return x == ref and math.copysign(1.0, x) == math.copysign(1.0, ref)
    return abs(x - ref) <= 1e-12 * abs(ref)


def test_special_values_match_the_reference():
    """Non-finite and extreme inputs (tests/golden/special_values.json, made
    by running the reference: oracle/gen_special.py): the reference starts
    every float sum at a[0,0] - a[0,0], so a non-finite a[0,0] gives NaN
    where the algebra gives +-inf; overflow, underflow and Ryser's signed
    zero follow the same arithmetic."""
    import json

    from conftest import GOLDEN

    cases = json.loads((GOLDEN / "special_values.json").read_text())
    for name, c in cases.items():
        vals = [[complex(x) for x in r] for r in c["matrix"]]  # repr() strings: '-inf', '(inf+1j)', ...
        a = np.array(vals) if c["complex"] else np.array([[z.real for z in r] for r in vals])
        for alg in ("combinatoric", "ryser", "glynn"):
            v = getattr(P, alg)(a)
            ref = complex(c[alg])
            if c["complex"]:
                ok = _same_special(v.real, ref.real) and _same_special(v.imag, ref.imag)
            else:
                ok = _same_special(float(v), ref.real)
            assert ok, (name, alg, v, c[alg])


def test_batch_from_pinned_host_memory():
    """A page-locked host batch (pinned torch tensor) is read by the DMA in
    place (no staging copy): same values as the pageable path, chunked
    pipeline included (batch larger than one 32 MB chunk)."""
    import torch

    rng = np.random.default_rng(12)
    a = rng.standard_normal((70_000, 8, 8)) / np.sqrt(8)  # 35.8 MB: two chunks
    want = P.opt_batch(a)
    t = torch.from_numpy(a).pin_memory()
    assert t.is_pinned()
    got = P.opt_batch(t)
    assert np.array_equal(np.asarray(got), want)
    r = rng.standard_normal((1000, 4, 10)) / np.sqrt(10)
    assert np.array_equal(np.asarray(P.opt_batch(torch.from_numpy(r).pin_memory())), P.opt_batch(r))


def test_batch_from_partly_registered_host_memory():
    """cudaHostRegister over only the first half of a host batch: the array
    is not page-locked end to end, so it takes the staged route (the DMA
    never reads past the registered range) and gives the same values."""
    import torch

    rng = np.random.default_rng(13)
    a = rng.standard_normal((70_000, 8, 8)) / np.sqrt(8)
    want = P.opt_batch(a)
    rt = torch.cuda.cudart()
    half = (a.nbytes // 2) & ~4095
    assert int(rt.cudaHostRegister(a.ctypes.data, half, 0)) == 0
    try:
        got = P.opt_batch(a)
    finally:
        rt.cudaHostUnregister(a.ctypes.data)
    assert np.array_equal(got, want)
