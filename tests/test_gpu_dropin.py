"""Drop-in corners on the GPU: CUDA tensors read in place, columns past the
walks' 62 (combinatoric and rectangular Ryser have no column cap in the
reference), ryser_rectangular on square integer matrices (the reference's
combination-order overflow flag), and opt's integer dispatch."""
from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2510_03421_b200 as P
from conftest import GOLDEN, decode_matrix
from oracle import oracle as O
from paper_2510_03421_b200.core import as_matrix, is_device

pytestmark = pytest.mark.gpu


def test_cuda_tensor_stays_on_device(rng):
    torch = pytest.importorskip("torch")
    a = rng.uniform(-1, 1, (16, 16))
    t = torch.tensor(a, device="cuda")
    mat = as_matrix(t)
    assert is_device(mat) and mat.data.is_cuda and mat.data.data_ptr() != t.data_ptr()  # private copy
    ref = P.glynn(a)
    assert P.glynn(t) == pytest.approx(ref, rel=1e-13)
    assert P.ryser(t) == pytest.approx(ref, rel=1e-10)
    assert P.opt(t) == pytest.approx(ref, rel=1e-10)
    assert P.glynn(t.T) == pytest.approx(P.glynn(a.T), rel=1e-13)
    tall = torch.tensor(rng.uniform(-1, 1, (9, 5)), device="cuda")  # m > n: transposed on the device
    assert P.ryser(tall) == pytest.approx(P.ryser(tall.cpu().numpy()), rel=1e-12)
    c = torch.tensor(rng.uniform(-1, 1, (10, 10)) + 1j * rng.uniform(-1, 1, (10, 10)), device="cuda")
    assert P.glynn(c) == pytest.approx(P.glynn(c.cpu().numpy()), rel=1e-13)
    i = torch.tensor(rng.integers(-3, 4, (9, 9)), device="cuda")
    exact = O.exact_int128("ryser", i.cpu().numpy())
    assert P.glynn(i) == exact and P.ryser(i) == exact and P.combinatoric(i) == exact
    assert P.glynn(i.to(torch.int32)) == exact
    b = torch.tensor(rng.random((8, 8)) < 0.5, device="cuda")  # bool -> int64 on the device
    assert P.opt(b) == O.exact_int128("glynn", b.cpu().numpy().astype(np.int64))
    with pytest.raises(TypeError):
        P.glynn(torch.zeros(3, device="cuda"))
    with pytest.raises(ValueError):
        P.glynn(torch.zeros((0, 3), device="cuda"))


def test_columns_past_62():
    """The reference caps only its Gray walks at 62 columns
    (src/algorithms.py:47, 148, 171); combinatoric and ryser_rect take any
    width (src/algorithms.py:71-90, 118-137)."""
    assert P.combinatoric(np.ones((1, 100), dtype=np.int64)) == 100
    assert P.ryser(np.ones((2, 70), dtype=np.int64)) == 70 * 69
    assert P.ryser_rectangular(np.ones((2, 70))) == pytest.approx(70 * 69, rel=1e-15)
    assert P.opt(np.ones((2, 70), dtype=np.int64)) == 70 * 69
    assert P.opt(np.ones((2, 70))) == pytest.approx(70 * 69, rel=1e-15)
    g = np.random.default_rng(70)
    for m, n in ((1, 200), (2, 90), (3, 64), (4, 66)):
        a = g.integers(-3, 4, (m, n)).astype(np.int64)
        ref = O.brute_force(a.tolist()) if math.perm(n, m) <= 3e5 else O.permanent("combinatoric", a)[0]
        assert P.combinatoric(a) == ref, (m, n)
        assert P.ryser(a) == ref, (m, n)
        f = g.uniform(-1, 1, (m, n))
        cf = P.combinatoric(f)
        assert P.ryser(f) == pytest.approx(cf, rel=1e-12, abs=1e-12 * math.perm(n, m) ** 0.5)
    with pytest.raises(ValueError):  # the Gray walks keep the reference's cap
        P.glynn(np.ones((2, 70)))
    with pytest.raises(ValueError):
        P.ryser(np.ones((63, 63)))


def test_ryser_rectangular_square_int_flags(ref_int_walk):
    """ryser_rectangular on a square integer matrix runs the reference's
    ryser_rect_int (combination order): value and overflow flag equal the
    oracle's restatement of that kernel, near the int64 onset too."""
    for case in ref_int_walk:
        a = decode_matrix(case["matrix"])
        if a.shape[0] != a.shape[1]:
            continue
        val, ovf = O.kernel("ryser_rect", a)
        got = P.permanent_ryser_rectangular(as_matrix(a))
        assert got.overflowed == ovf, a.shape
        if not ovf:
            assert got.value == val == int(case["exact"])


def test_opt_integer_dispatch_matches_reference():
    """opt on integers selects with the reference's table, so OverflowError
    appears exactly where the reference's opt raises it."""
    a = np.full((6, 6), 300, dtype=np.int64)
    assert P.opt(a) == 524880000000000000 == math.factorial(6) * 300 ** 6
    near = [decode_matrix(c["matrix"]) for c in __import__("json").loads((GOLDEN / "ref_int_walk.json").read_text())]
    from paper_2510_03421_b200.dispatch import default_params, select_algorithm

    for a in near:
        alg = select_algorithm(*a.shape, default_params())
        exp = O.permanent(alg.value, a)
        try:
            assert P.opt(a) == exp[0] and not exp[1]
        except OverflowError:
            assert exp[1]
