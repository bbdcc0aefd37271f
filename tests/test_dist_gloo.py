"""Multi-process (world_size 2, gloo, CPU) coverage of the sharded path:
range planning, the all-gather of raw partials, and the ordered combine +
normalization -- with the CPU oracle's range walk standing in for the GPU
kernel (partial_fn), so no device is needed."""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_partial(alg, a, k0, k1):
    sys.path.insert(0, str(ROOT))
    from oracle import oracle as O

    setup = O.walk_setup(alg, a)
    if np.iscomplexobj(a):
        (rh, rl), (ih, il) = O.walk_dd_mt(setup, k0, k1, nthreads=1)
        return [rh, rl, ih, il, 0, 0, 0, 0]
    (rh, rl), _ = O.walk_dd_mt(setup, k0, k1, nthreads=1)
    return [rh, rl, 0, 0, 0, 0, 0, 0]


def oracle_int_partial(alg, a, k0, k1):
    """Exact int128 range sum from the oracle, packed as the engine's
    width-128 partial (the finish then uses the a-priori fit certificate)."""
    sys.path.insert(0, str(ROOT))
    from oracle import oracle as O
    from paper_2510_03421_b200.sharded import int128_partial

    return int128_partial(O.walk_i128_mt(O.walk_setup(alg, a), k0, k1, nthreads=1))


def _worker(rank, world, port, cases, q):
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_03421_b200.sharded import sharded_permanent

    out = []
    for alg, a in cases:
        if a.dtype.kind == "i":
            out.append(sharded_permanent(a, alg=alg, partial_fn=oracle_int_partial, exact="int128"))
        else:
            out.append(sharded_permanent(a, alg=alg, partial_fn=oracle_partial))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_combine_gloo(world):
    from oracle import oracle as O

    g = np.random.default_rng(7)
    cases = [("glynn", g.uniform(-1, 1, (11, 11))), ("ryser", g.uniform(-1, 1, (10, 10))),
             ("glynn", g.uniform(-1, 1, (9, 9)) + 1j * g.uniform(-1, 1, (9, 9))),
             ("ryser", g.uniform(-1, 1, (4, 9))), ("glynn", g.uniform(-1, 1, (3, 3))),
             ("glynn", g.integers(-2, 3, (10, 10))), ("ryser", g.integers(0, 2, (9, 9))),
             ("ryser", g.integers(-3, 4, (5, 9))), ("glynn", g.integers(0, 5, (4, 7)))]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, (alg, a) in enumerate(cases):
        vals = [results[r][i] for r in range(world)]
        if a.dtype.kind == "i":
            assert all(v == vals[0] for v in vals)
            assert vals[0] == O.exact_int128("ryser", a)  # exact (oracle int128 walk)
            continue
        ref = O.permanent("ryser", a)[0]
        assert all(v == vals[0] for v in vals)  # identical on every rank
        assert abs(vals[0] - ref) <= 1e-12 * max(1.0, abs(ref))


def oracle_batch(part):
    sys.path.insert(0, str(ROOT))
    from oracle import oracle as O

    return [O.permanent("glynn", x)[0] for x in part]


def _batch_worker(rank, world, port, batches, q):
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_03421_b200.sharded import sharded_batch

    q.put((rank, [sharded_batch(A, batch_fn=oracle_batch) for A in batches]))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_batch_gloo():
    """Batch split over 3 ranks (ragged slices), one all-gather: every rank
    holds the whole result in batch order."""
    from oracle import oracle as O

    g = np.random.default_rng(11)
    batches = [g.uniform(-1, 1, (10, 5, 5)), g.uniform(-1, 1, (7, 4, 4)) + 1j * g.uniform(-1, 1, (7, 4, 4)),
               g.uniform(-1, 1, (2, 3, 3))]
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, batches, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, A in enumerate(batches):
        ref = np.array([O.permanent("glynn", x)[0] for x in A])
        for r in range(world):
            assert results[r][i].shape == (A.shape[0],)
            np.testing.assert_array_equal(results[r][i], ref)
