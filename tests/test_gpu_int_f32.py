"""The FP32-quad exact int128 walk (csrc/int_walk32.cuh) against the oracle's
exact integer permanents and against the FP64-exact walk, bit for bit.
Needs a B200.

The walk is chosen by the host whenever the state entries group into quads
with bound products < 2^23 (engine_int.cu int_f32_quads); which kernel ran
is read from the est_kind slot of ``perm_walk_partial_i64``'s partial
(3 = FP32 estimate / integer upper levels, 4 = FP64 upper levels, 1 = the
FP64-exact walk of int_walk.cuh)."""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2510_03421_b200 as P
from conftest import GOLDEN
from oracle import oracle as O
from paper_2510_03421_b200 import sharded as S
from paper_2510_03421_b200 import workloads as W

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def est_kind(alg, a):
    m, n = a.shape
    steps = 1 << (n - 1 if alg == "glynn" else n)
    return int(S.gpu_partial_int(alg, a, 0, steps, exact="int128")[5])


def cases():
    rng = np.random.default_rng(20251021)
    out = []
    # every quad count 3..5 (n = 9..18), odd and even, 0/1 and signed
    for n in (9, 10, 11, 12, 13, 15, 16, 17, 18):
        out.append(("01", rng.integers(0, 2, (n, n)).astype(np.int64)))
        out.append(("pm2", rng.integers(-2, 3, (n, n)).astype(np.int64)))
    return out


@pytest.mark.parametrize("alg", ["glynn", "ryser"])
def test_f32_walk_matches_oracle(alg):
    ran = set()
    for kind, a in cases():
        want = O.exact_int128(alg, a)
        assert getattr(P, alg)(a, exact="int128") == want, (kind, a.shape)
        ran.add(est_kind(alg, a))
    assert 4 in ran, ran  # the FP64-upper-level variant ran


def test_integer_upper_levels_variant():
    """Quads between 2^21 and 2^23: the four-quad products pass 2^84, so the
    96-bit products come from the integer multiplies (est_kind 3)."""
    rng = np.random.default_rng(5)
    kinds = set()
    for n in (14, 16):
        for _ in range(3):
            a = rng.integers(-5, 6, (n, n)).astype(np.int64)
            for alg in ("glynn", "ryser"):
                assert getattr(P, alg)(a, exact="int128") == O.exact_int128(alg, a), (alg, n)
                kinds.add(est_kind(alg, a))
    assert 3 in kinds, kinds


def test_large_entries_keep_the_fp64_exact_walk():
    """Column bounds past 2^23 / 4 per quad: not eligible, and still exact."""
    rng = np.random.default_rng(6)
    a = rng.integers(-300, 301, (12, 12)).astype(np.int64)
    assert est_kind("glynn", a) in (0, 1, 2)
    assert P.glynn(a, exact="int128") == O.exact_int128("glynn", a)


def test_rectangular_glynn_int128():
    """Ones-padded rectangular Glynn (pad rows flip too) through the quad walk."""
    rng = np.random.default_rng(8)
    for m, n in ((8, 12), (10, 13), (6, 16)):
        a = rng.integers(-2, 3, (m, n)).astype(np.int64)
        assert P.glynn(a, exact="int128") == O.exact_int128("glynn", a), (m, n)


def test_c4_configs_match_fixture_and_fp64_walk():
    """C4a / C4b through the quad walk equal the committed exact values; the
    FP64-exact walk (PERM_INT_F32=0, read at first use, so a subprocess) gives
    the same bits."""
    fix = json.load(open(GOLDEN / "c4.json"))
    a, b = W.c4a(), W.c4b()
    va, vb = P.glynn(a, exact="int128"), P.glynn(b, exact="int128")
    assert str(va) == fix["c4a_exact"] and str(vb) == fix["c4b_exact"]
    assert est_kind("glynn", a) == 4 and est_kind("glynn", b) in (3, 4)
    assert P.ryser(b, exact="int128") == vb
    code = ("import sys; sys.path.insert(0, '.'); import paper_2510_03421_b200 as P; "
            "from paper_2510_03421_b200 import workloads as W; "
            "print(P.glynn(W.c4b(), exact='int128'))")
    env = dict(os.environ, PERM_INT_F32="0")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert int(r.stdout.strip().splitlines()[-1]) == vb


def test_sharded_ranges_sum_to_the_whole():
    """Unaligned shard boundaries (world 3) through the partial / finish protocol."""
    a = W.c4b()[:20, :20].copy()
    want = O.exact_int128("glynn", a)
    assert S.sharded_permanent(a, alg="glynn", exact="int128") == want
    m, n = a.shape
    for alg in ("glynn", "ryser"):
        parts = [S.gpu_partial_int(alg, a, *S.shard_range(alg, m, n, r, 3), exact="int128") for r in range(3)]
        assert {int(p[5]) for p in parts} <= {3, 4}
        assert S.finish_int(alg, a, np.stack(parts), exact="int128") == want
