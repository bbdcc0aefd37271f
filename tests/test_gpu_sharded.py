"""Sharded walks on the GPU: exact-integer shards (checked int64 with the
reference's overflow flag across shards, certified int128), the
single-process multi-device driver (perm_sharded_*; here with one device
listed several times), and the NCCL path for integers."""
from __future__ import annotations

import json

import numpy as np
import pytest

import paper_2510_03421_b200 as P
from conftest import GOLDEN, decode_matrix
from oracle import oracle as O
from paper_2510_03421_b200 import sharded as S
from paper_2510_03421_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _shards_int(alg, a, world, exact):
    m, n = a.shape
    parts = [S.gpu_partial_int(alg, a, *S.shard_range(alg, m, n, r, world), exact=exact) for r in range(world)]
    return S.finish_int(alg, a, np.stack(parts), exact=exact)


@pytest.fixture(scope="module")
def near_overflow():
    return json.loads((GOLDEN / "ref_int_walk.json").read_text())


@pytest.mark.parametrize("world", [1, 2, 3, 4, 7])
def test_checked_int_shards_keep_reference_flags(near_overflow, world):
    """The rank-ordered combine of (sum, min/max prefix, flag) summaries
    raises OverflowError exactly where the reference's sequential checked
    walk does, for every shard count."""
    for case in near_overflow:
        a = decode_matrix(case["matrix"])
        exact = int(case["exact"])
        for alg, r in case["results"].items():
            if alg == "ryser" and a.shape[0] < a.shape[1]:
                continue
            if r["overflowed"]:
                with pytest.raises(OverflowError):
                    _shards_int(alg, a, world, None)
            else:
                assert _shards_int(alg, a, world, None) == exact
            assert _shards_int(alg, a, world, "int128") == exact


def test_int128_shards_c4():
    c4 = json.loads((GOLDEN / "c4.json").read_text())
    assert _shards_int("glynn", W.c4b(), 4, "int128") == int(c4["c4b_exact"])
    assert _shards_int("ryser", W.c4b(), 3, "int128") == int(c4["c4b_exact"])
    a = W.c4a()[:24, :24]
    ref = O.exact_int128("glynn", a)
    for world in (2, 5):
        assert _shards_int("glynn", a, world, "int128") == ref
        assert _shards_int("ryser", a, world, "int128") == ref


def test_int_shard_edge_cases():
    big = np.array([[2**62, 3], [5, 2**62]], dtype=np.int64)   # 128-bit state kernel, empty shards
    for world in (1, 2, 4):
        assert _shards_int("glynn", big, world, "int128") == 2**124 + 15
        assert _shards_int("ryser", big, world, "int128") == 2**124 + 15
        with pytest.raises(OverflowError):
            _shards_int("glynn", big, world, None)
    rect = np.random.default_rng(5).integers(-3, 4, (6, 13)).astype(np.int64)
    ref = O.exact_int128("ryser", rect)
    for world in (1, 3, 8):
        assert _shards_int("glynn", rect, world, "int128") == ref
        assert _shards_int("ryser", rect, world, "int128") == ref
        assert _shards_int("glynn", rect, world, None) == ref
    with pytest.raises(ValueError):  # checked rect Ryser follows the combination order: no Gray shards
        _shards_int("ryser", rect, 2, None)
    # ... so sharded_permanent evaluates it whole on every rank (world of one here)
    assert P.sharded_permanent(rect, alg="ryser") == ref
    with pytest.raises(ValueError):  # partial of the other width
        p = S.gpu_partial_int("glynn", rect, 0, 1 << 12, exact=None)
        S.finish_int("glynn", rect, p[None, :], exact="int128")


def test_multi_device_driver():
    """perm_sharded_*: shards on a device list from one process (one GPU
    listed several times here), identical to the single-device call."""
    a = W.c5(26)
    ref = P.glynn(a)
    for devs in ((0,), (0, 0), (0, 0, 0, 0, 0)):
        v = P.multi_device_permanent(a, devices=devs)
        assert v == pytest.approx(ref, rel=1e-13)
    v, M = P.multi_device_permanent(W.c3a(), devices=(0, 0, 0), mag=True)
    assert abs(v - P.glynn(W.c3a())) <= 1e-12 * M
    r = P.multi_device_permanent(W.c5(22), alg="ryser", devices=(0, 0))
    assert r == pytest.approx(P.ryser(W.c5(22)), rel=1e-10)
    c4 = json.loads((GOLDEN / "c4.json").read_text())
    assert P.multi_device_permanent(W.c4b(), devices=(0, 0, 0), exact="int128") == int(c4["c4b_exact"])
    small = np.random.default_rng(2).integers(-2, 3, (12, 12)).astype(np.int64)
    assert P.multi_device_permanent(small, devices=(0, 0)) == O.exact_int128("ryser", small)
    with pytest.raises(OverflowError):
        P.multi_device_permanent(np.array([[2**31, 1], [1, 2**31]], dtype=np.int64), devices=(0, 0))
    with pytest.raises(ValueError):
        P.multi_device_permanent(a, devices=())


def test_multi_device_driver_nccl_exchange(monkeypatch):
    """perm_sharded_* with the NCCL exchange (ncclCommInitAll over the device
    list + one grouped ncclAllGather of the 8-double partials), forced on a
    single-device list here; results identical to the host exchange."""
    a = W.c5(24)
    monkeypatch.setenv("PERM_SHARDED_EXCHANGE", "host")
    host = P.multi_device_permanent(a, devices=(0,))
    monkeypatch.setenv("PERM_SHARDED_EXCHANGE", "nccl")
    import ctypes as C

    from paper_2510_03421_b200 import _lib

    assert _lib.load().perm_sharded_exchange(1, (C.c_int * 1)(0)) == 1  # libnccl loaded: NCCL path
    assert _lib.load().perm_sharded_exchange(2, (C.c_int * 2)(0, 0)) == 0  # duplicate device: host path
    for _ in range(2):  # second call reuses the cached communicator
        assert P.multi_device_permanent(a, devices=(0,)) == host
    c = W.c3b()[:14, :20]
    nccl = P.multi_device_permanent(c, devices=(0,))
    monkeypatch.setenv("PERM_SHARDED_EXCHANGE", "host")
    assert P.multi_device_permanent(c, devices=(0,)) == nccl
    assert P.multi_device_permanent(c, devices=(0, 0)) == pytest.approx(nccl, rel=1e-12)


def test_sharded_nccl_single_rank_int():
    import os
    import socket

    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        c4 = json.loads((GOLDEN / "c4.json").read_text())
        assert P.sharded_permanent(W.c4b(), exact="int128") == int(c4["c4b_exact"])
        small = np.random.default_rng(4).integers(0, 3, (11, 11)).astype(np.int64)
        assert P.sharded_permanent(small, alg="ryser") == O.exact_int128("ryser", small)
        A = W.c1()
        np.testing.assert_array_equal(P.sharded_batch(A), P.opt_batch(A))
    finally:
        dist.destroy_process_group()


def _range_case(alg, a, span=1 << 22):
    """GPU raw partial over the last `span` indices of the walk (seeded from
    high Gray bits) vs the oracle's double-double walk over the same range."""
    m, n = a.shape
    total = (1 << (n - 1)) if alg == "glynn" else (1 << n)
    span = min(span, total // 4)
    k0, k1 = total - span, total
    part = S.gpu_partial(alg, a, k0, k1, mag=True)
    setup = O.walk_setup(alg, a)
    (rh, rl), (ih, il) = O.walk_dd_mt(setup, k0, k1)
    gpu = complex(part[0] + part[1], part[2] + part[3])
    ref = complex(rh + rl, ih + il)
    return abs(gpu - ref) / max(part[4], 1e-300)


@pytest.mark.parametrize("n", list(range(17, 53)) + [56, 62])
def test_walk_kernels_every_state_length(n):
    """Every real walk instantiation the C5 n-sweep can reach (P = 17..52 hold
    U[0] in registers; 56 and 62 do not), on a 2^22-step range at the end of
    the walk: square Glynn (P = n, B = n-1) and square Ryser (P = B = n)."""
    rng = np.random.default_rng(1000 + n)
    a = rng.uniform(-1, 1, (n, n)) / n
    assert _range_case("glynn", a) <= 1e-11
    assert _range_case("ryser", a) <= 1e-11


@pytest.mark.parametrize("m,n", [(17, 23), (24, 27), (30, 33), (36, 39)])
def test_weighted_walk_kernels(m, n):
    """Rectangular Ryser: popcount-weighted walk with P = m state rows."""
    rng = np.random.default_rng(m * 100 + n)
    a = rng.uniform(-1, 1, (m, n)) / n
    assert _range_case("ryser", a) <= 1e-11


@pytest.mark.parametrize("n", [20, 24, 28, 32])
def test_complex_walk_kernels(n):
    rng = np.random.default_rng(7 * n)
    a = (rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))) / n
    assert _range_case("glynn", a) <= 1e-11
