"""The C ABI library: it loads, exports exactly what include/permanent_b200.h
declares, and its pure-host entry points (sharding plan, partial combine,
dispatch) behave.  No compute call is made on CPU except to check that the
product path fails loudly without a GPU (there is no CPU fallback)."""
from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2510_03421_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "permanent_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(perm_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    for must in ("perm_glynn_f64", "perm_glynn_c128", "perm_ryser_f64", "perm_ryser_c128",
                 "perm_comb_f64", "perm_comb_c128", "perm_comb_i64", "perm_glynn_i64",
                 "perm_ryser_i64", "perm_walk_partial_f64", "perm_walk_finish_f64", "perm_select",
                 "perm_batch_f64", "perm_batch_c128"):
        assert must in syms, must


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (perm_[a-z0-9_]+)", out))
    for s in declared_symbols():
        assert s in exported, s
        assert hasattr(lib, s)
    # and the Python binding table covers the header
    assert set(declared_symbols()) <= set(_lib.SIGNATURES)


def test_version_and_select():
    lib = _lib.load()
    assert lib.perm_version() >= 100
    p = (C.c_double * 8)(-1.0, -0.105, 1.655, 5.0, 1.0, -0.007, -0.199, 13.0)
    assert lib.perm_select(3, 3, p, 0, 0) == _lib.ALG_COMBINATORIC
    assert lib.perm_select(20, 20, p, 0, 0) == _lib.ALG_GLYNN
    assert lib.perm_select(4, 20, p, 0, 0) == _lib.ALG_RYSER


def test_batch_select():
    """Batch dispatch: the 4+4 Laplace formula for 8x8 (4), the partition
    formula (3) for m <= 4 < n and m = 5, 6 with n >= m + 2, Glynn for other
    squares and for the remaining rectangles with n >= 9, Ryser otherwise."""
    lib = _lib.load()
    assert lib.perm_batch_select(8, 8) == 4
    assert lib.perm_batch_select(4, 10) == 3
    assert lib.perm_batch_select(1, 16) == 3
    assert lib.perm_batch_select(5, 5) == _lib.ALG_GLYNN
    assert lib.perm_batch_select(5, 9) == 3
    assert lib.perm_batch_select(5, 6) == _lib.ALG_RYSER
    assert lib.perm_batch_select(6, 8) == 3
    assert lib.perm_batch_select(6, 7) == _lib.ALG_RYSER
    assert lib.perm_batch_select(7, 8) == _lib.ALG_RYSER
    assert lib.perm_batch_select(7, 12) == _lib.ALG_GLYNN
    assert lib.perm_batch_select(12, 16) == _lib.ALG_GLYNN


@pytest.mark.parametrize("alg,m,n", [(2, 36, 36), (2, 20, 28), (1, 30, 30), (1, 5, 33), (2, 3, 3)])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 7, 8])
def test_shards_partition_the_walk(alg, m, n, world):
    lib = _lib.load()
    steps = lib.perm_walk_steps(alg, m, n)
    assert steps == (1 << (n - 1) if alg == 2 else 1 << n)
    prev = 0
    for r in range(world):
        b, e = C.c_uint64(), C.c_uint64()
        assert lib.perm_walk_shard(alg, m, n, r, world, C.byref(b), C.byref(e)) == _lib.OK
        assert b.value == prev and e.value >= b.value
        prev = e.value
    assert prev == steps


def test_finish_combines_partials_in_order():
    """Double-double combine + Glynn normalization of raw partials."""
    lib = _lib.load()
    a = np.eye(4)
    parts = np.zeros((3, 8))
    parts[:, 0] = [1.0, 2.0**-60, 7.0]  # hi parts
    out = (C.c_double * 2)()
    mg = C.c_double()
    st = lib.perm_walk_finish_f64(2, 4, 4, C.c_void_p(a.ctypes.data), 4, C.c_void_p(parts.ctypes.data), 3,
                                  out, C.byref(mg))
    assert st == _lib.OK
    assert out[0] == (8.0 + 2.0**-60) / 8.0


def test_bad_shapes_rejected_by_the_abi():
    lib = _lib.load()
    b, e = C.c_uint64(), C.c_uint64()
    assert lib.perm_walk_shard(2, 5, 3, 0, 1, C.byref(b), C.byref(e)) == _lib.BAD_SHAPE
    assert lib.perm_walk_shard(2, 3, 63, 0, 1, C.byref(b), C.byref(e)) == _lib.BAD_SHAPE
    assert lib.perm_walk_shard(2, 3, 3, 2, 2, C.byref(b), C.byref(e)) == _lib.BAD_ARG


def _int_plan(alg, a):
    lib = _lib.load()
    a = np.ascontiguousarray(a, dtype=np.int64)
    kind, groups = C.c_int(-1), C.c_int(-1)
    st = lib.perm_int_walk_plan(alg, a.shape[0], a.shape[1], a.ctypes.data, a.shape[1], C.byref(kind),
                                C.byref(groups))
    return st, kind.value, groups.value


def test_int_walk_plan_is_host_only_and_follows_the_entry_bounds():
    """Which exact int128 walk a matrix takes is decided on the host from its
    column bounds (no CUDA call): C4a / C4b-like matrices take the quad walk,
    entries past the 23-bit quad / 51-bit group bounds the generic 128-bit
    state, the weighted (rectangular Ryser) walk always the generic one."""
    rng = np.random.default_rng(1)
    c4a = rng.integers(0, 2, (32, 32))
    c4b = rng.integers(-2, 3, (28, 28))
    for alg in (1, 2):
        st, kind, groups = _int_plan(alg, c4a)
        assert st == _lib.OK and kind in (3, 4) and groups == 8
    st, kind, groups = _int_plan(2, c4b)
    assert st == _lib.OK and kind in (3, 4) and groups == 7
    # the plan depends on the bounds only, not on the values
    assert _int_plan(2, c4a) == _int_plan(2, np.ones((32, 32)))
    assert _int_plan(2, rng.integers(-(10**12), 10**12, (24, 24))) == (_lib.OK, 0, 0)
    assert _int_plan(2, rng.integers(-3, 3, (6, 6))) == (_lib.OK, 0, 0)  # below 8 Gray bits
    assert _int_plan(1, rng.integers(-3, 3, (10, 20))) == (_lib.OK, 0, 0)  # weighted walk
    st, kind, groups = _int_plan(2, rng.integers(-3, 3, (10, 20)))  # padded Glynn: 20 state entries
    assert st == _lib.OK and kind in (3, 4) and groups == 5
    assert _int_plan(2, np.ones((5, 3)))[0] == _lib.BAD_SHAPE
    lib = _lib.load()
    assert lib.perm_int_walk_plan(2, 3, 3, None, 3, None, None) == _lib.BAD_ARG


def test_int_walk_plan_quads_can_be_switched_off():
    code = (
        "import ctypes as C, numpy as np\n"
        "from paper_2510_03421_b200 import _lib\n"
        "lib = _lib.load(); a = np.ones((32, 32), dtype=np.int64)\n"
        "k, g = C.c_int(), C.c_int()\n"
        "assert lib.perm_int_walk_plan(2, 32, 32, a.ctypes.data, 32, C.byref(k), C.byref(g)) == 0\n"
        "print(k.value, g.value)\n"
    )
    import os
    import sys

    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env={**os.environ, "PERM_INT_F32": "0"},
                         capture_output=True, text=True, check=True).stdout.split()
    assert int(out[0]) == 1 and int(out[1]) >= 1  # FP64-exact groups


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2510_03421_b200 as P

    with pytest.raises(_lib.EngineUnavailable):
        P.glynn(np.random.default_rng(0).uniform(-1, 1, (5, 5)))


def test_batch_shape_contracts_without_gpu():
    """Shape validation of the batch entry points happens before any device
    work, so it is exercised here: the partition formula stops at m = 6
    (complex m = 5) and n = 62, the Laplace formula is 8x8 only,
    Glynn batches stop at n = 30, the other algorithms at n = 16."""
    import numpy as np

    import paper_2510_03421_b200 as P

    with pytest.raises(ValueError):
        P.partition_batch(np.zeros((2, 7, 9)))
    with pytest.raises(ValueError):
        P.laplace_batch(np.zeros((2, 6, 6)))
    with pytest.raises(ValueError):
        P.ryser_batch(np.zeros((2, 17, 17)))
    with pytest.raises(ValueError):
        P.glynn_batch(np.zeros((2, 31, 31)))
    with pytest.raises(ValueError):
        P.opt_batch(np.zeros((2, 7, 31)))  # m >= 7 rectangles: batched walks stop at n = 30
    with pytest.raises(ValueError):
        P.partition_batch(np.zeros((2, 5, 63)))  # 62 columns at most
    with pytest.raises(ValueError):
        P.partition_batch(np.zeros((2, 6, 20)) + 0j)  # complex: m <= 5
