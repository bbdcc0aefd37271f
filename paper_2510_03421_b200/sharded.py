"""One large permanent sharded over torch.distributed ranks.

The Gray index space of the walk ([0, 2^(n-1)) for Glynn, [0, 2^n) for Ryser)
is cut into ``world`` contiguous, power-of-two-aligned ranges
(``perm_walk_shard``); rank r walks its range on its own GPU and produces a
compensated partial (re_hi, re_lo, im_hi, im_lo, M).  The only exchange is one
all-gather of those 8 doubles per rank (NCCL over NVLink/NVSwitch for CUDA
tensors, gloo for CPU tensors), after which every rank combines the partials
in rank order with a double-double sum and applies the normalization
(``perm_walk_finish``) -- deterministic, and exact to the last bit across
ranks.  The reference has no counterpart (sharding is a SPEC.md:274 non-goal).

Integer matrices take the exact path: each rank's partial is 8 int64
(``perm_walk_partial_i64``): for ``exact=None`` the checked-int64 summary
(sum, min/max running prefix, flag) whose rank-ordered combine reproduces the
reference's OverflowError exactly, for ``exact="int128"`` the range's sum
mod 2^128 plus its FP64 estimate for the fit certificate.

``multi_device_permanent`` is the single-process form: one call, shards on
a list of local devices (``perm_sharded_*``).

``partial_fn`` lets tests substitute a CPU walk for the GPU kernel so the
multi-process logic runs under gloo without a device.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

ALG = {"glynn": _lib.ALG_GLYNN, "ryser": _lib.ALG_RYSER}


def shard_range(alg: str, m: int, n: int, rank: int, world: int):
    lib = _lib.load()
    b, e = C.c_uint64(), C.c_uint64()
    _lib.check(lib.perm_walk_shard(ALG[alg], m, n, rank, world, C.byref(b), C.byref(e)), "shard")
    return int(b.value), int(e.value)


def gpu_partial(alg: str, a: np.ndarray, k0: int, k1: int, mag: bool = False, device_out=None, stream=None):
    """Raw partial over [k0, k1) on the current GPU.  With ``device_out`` (a
    float64 CUDA tensor of 8) the call is asynchronous on ``stream``."""
    lib = _lib.load()
    a = np.ascontiguousarray(a)
    cplx = np.iscomplexobj(a)
    m, n = a.shape
    fn = lib.perm_walk_partial_c128 if cplx else lib.perm_walk_partial_f64
    if device_out is not None:
        st = fn(ALG[alg], m, n, C.c_void_p(a.ctypes.data), n, 0, k0, k1, int(mag),
                C.c_void_p(device_out.data_ptr()), 1, C.c_void_p(stream) if stream else None)
        _lib.check(st, "partial")
        return device_out
    out = np.zeros(8)
    st = fn(ALG[alg], m, n, C.c_void_p(a.ctypes.data), n, 0, k0, k1, int(mag), C.c_void_p(out.ctypes.data), 0,
            None)
    _lib.check(st, "partial")
    return out


def finish(alg: str, a: np.ndarray, partials: np.ndarray):
    """Combine [G, 8] raw partials in order and normalize -> (value, M)."""
    lib = _lib.load()
    a = np.ascontiguousarray(a)
    cplx = np.iscomplexobj(a)
    m, n = a.shape
    parts = np.ascontiguousarray(partials, dtype=np.float64).reshape(-1, 8)
    out = (C.c_double * 2)()
    mg = C.c_double()
    fn = lib.perm_walk_finish_c128 if cplx else lib.perm_walk_finish_f64
    _lib.check(fn(ALG[alg], m, n, C.c_void_p(a.ctypes.data), n, C.c_void_p(parts.ctypes.data), parts.shape[0],
                  out, C.byref(mg)), "finish")
    return (complex(out[0], out[1]) if cplx else float(out[0])), mg.value


_TAG128 = 0x7065726d31323800  # perm_walk_partial_i64's width-128 tag


def _width(exact) -> int:
    if exact is None:
        return 64
    if exact == "int128":
        return 128
    raise ValueError(f"exact must be None or 'int128', got {exact!r}")


def _int_status(st: int, what: str):
    if st == _lib.OVERFLOW:
        raise OverflowError(f"{what}: {_lib.last_error()}")
    _lib.check(st, what)


def gpu_partial_int(alg: str, a: np.ndarray, k0: int, k1: int, exact=None) -> np.ndarray:
    """Exact-integer partial (8 int64) over [k0, k1) on the current GPU."""
    lib = _lib.load()
    a = np.ascontiguousarray(a, dtype=np.int64)
    m, n = a.shape
    out = np.zeros(8, np.int64)
    st = lib.perm_walk_partial_i64(ALG[alg], m, n, C.c_void_p(a.ctypes.data), n, 0, _width(exact), k0, k1,
                                   out.ctypes.data_as(C.POINTER(C.c_int64)), None)
    _lib.check(st, "int partial")
    return out


def int128_partial(raw: int) -> np.ndarray:
    """Pack an exact range sum (a CPU walk standing in for the kernel, tests
    only) as a width-128 partial without FP64 estimate; its finish then
    relies on the a-priori fit certificate."""
    r = raw % (1 << 128)
    lo, hi = r & ((1 << 64) - 1), r >> 64
    v = np.zeros(8, np.int64)
    v[0] = np.array(lo, dtype=np.uint64).view(np.int64)
    v[1] = np.array(hi, dtype=np.uint64).view(np.int64)
    v[7] = _TAG128
    return v


def _to_int(out) -> int:
    lo, hi = int(out[0]) & ((1 << 64) - 1), int(out[1])
    return (hi << 64) | lo


def finish_int(alg: str, a: np.ndarray, partials: np.ndarray, exact=None) -> int:
    """Combine [G, 8] integer partials in rank order -> the exact permanent;
    OverflowError where the reference's checked walk overflows (exact=None)
    or the int128 value is not certified (exact='int128')."""
    lib = _lib.load()
    a = np.ascontiguousarray(a, dtype=np.int64)
    m, n = a.shape
    parts = np.ascontiguousarray(partials, dtype=np.int64).reshape(-1, 8)
    out = (C.c_int64 * 2)()
    fits = C.c_int()
    st = lib.perm_walk_finish_i64(ALG[alg], m, n, C.c_void_p(a.ctypes.data), n, _width(exact),
                                  parts.ctypes.data_as(C.POINTER(C.c_int64)), parts.shape[0], out, C.byref(fits))
    _int_status(st, "int finish")
    return _to_int(out)


def _is_int(a: np.ndarray) -> bool:
    return a.dtype.kind in "iub"


def _world(group):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group), dist.get_backend(group)
    return 0, 1, None


def _gather(part, world, group):
    import torch
    import torch.distributed as dist

    if world == 1:
        return part.cpu().numpy()
    gathered = torch.empty(world * part.numel(), dtype=part.dtype, device=part.device)
    dist.all_gather_into_tensor(gathered, part, group=group)
    return gathered.cpu().numpy()


def _sharded_int(a, alg, group, exact, partial_fn):
    import torch

    a = np.ascontiguousarray(a, dtype=np.int64)
    m, n = a.shape
    rank, world, backend = _world(group)
    if alg == "ryser" and m < n and exact is None and partial_fn is None:
        # the checked-int64 flag of rectangular Ryser belongs to the
        # reference's sequential combination order (ryser_rect_int,
        # src/_kernels.py:265-365), not to a Gray range: every rank evaluates
        # it whole (combination-order kernel, sum_{s<=m} C(n, s) subsets --
        # the cheap form for the very rectangular shapes it is chosen for);
        # exact="int128" shards the Gray walk instead
        from . import engine

        value, ovf = engine.ryser_rect(a)
        if ovf:
            raise OverflowError("rectangular Ryser: an int64 intermediate overflowed (reference semantics)")
        return int(value)
    k0, k1 = shard_range(alg, m, n, rank, world)
    if partial_fn is not None:
        part = torch.tensor(np.asarray(partial_fn(alg, a, k0, k1), dtype=np.int64))
    else:
        part = torch.tensor(gpu_partial_int(alg, a, k0, k1, exact))
        if backend == "nccl":
            part = part.cuda()
    return finish_int(alg, a, _gather(part, world, group), exact)


def sharded_permanent(a, alg: str = "glynn", group=None, mag: bool = False, partial_fn=None, exact=None):
    """Permanent of one m x n matrix with its walk sharded over the ranks of
    ``group`` (default: the world).  Every rank returns the same value.
    float64 / complex128: returns (value, M) if ``mag`` else value.
    Integer matrices: the exact Python int (see module doc for ``exact``)."""
    import torch

    a = np.asarray(a)
    if a.shape[0] > a.shape[1]:
        a = a.T
    if _is_int(a):
        if mag:
            raise ValueError("mag is defined for float walks")
        return _sharded_int(a, alg, group, exact, partial_fn)
    a = np.ascontiguousarray(a, dtype=np.complex128 if np.iscomplexobj(a) else np.float64)
    m, n = a.shape
    rank, world, backend = _world(group)
    k0, k1 = shard_range(alg, m, n, rank, world)
    if partial_fn is not None:
        part = torch.tensor(np.asarray(partial_fn(alg, a, k0, k1), dtype=np.float64))
    elif backend == "nccl":
        part = torch.empty(8, dtype=torch.float64, device="cuda")
        gpu_partial(alg, a, k0, k1, mag, device_out=part, stream=torch.cuda.current_stream().cuda_stream)
    else:
        part = torch.tensor(gpu_partial(alg, a, k0, k1, mag))
    value, M = finish(alg, a, _gather(part, world, group))
    return (value, M) if mag else value


def multi_device_permanent(a, alg: str = "glynn", devices=(0,), mag: bool = False, exact=None):
    """One permanent with its walk split over local ``devices`` from this
    process (``perm_sharded_*``; a device may repeat).  Same results and
    return conventions as ``sharded_permanent``."""
    lib = _lib.load()
    a = np.asarray(a)
    if a.shape[0] > a.shape[1]:
        a = a.T
    devs = (C.c_int * len(devices))(*devices)
    if _is_int(a):
        a = np.ascontiguousarray(a, dtype=np.int64)
        m, n = a.shape
        out = (C.c_int64 * 2)()
        fits = C.c_int()
        st = lib.perm_sharded_i64(ALG[alg], m, n, C.c_void_p(a.ctypes.data), n, _width(exact), len(devices), devs,
                                  out, C.byref(fits))
        _int_status(st, "sharded int")
        return _to_int(out)
    cplx = np.iscomplexobj(a)
    a = np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)
    m, n = a.shape
    out = (C.c_double * 2)()
    mg = C.c_double()
    fn = lib.perm_sharded_c128 if cplx else lib.perm_sharded_f64
    _lib.check(fn(ALG[alg], m, n, C.c_void_p(a.ctypes.data), n, len(devices), devs, out,
                  C.byref(mg) if mag else None), "sharded")
    value = complex(out[0], out[1]) if cplx else float(out[0])
    return (value, mg.value) if mag else value


def batch_slice(B: int, rank: int, world: int):
    """Contiguous slice [b0, b1) of a batch of B matrices for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return B * rank // world, B * (rank + 1) // world


def sharded_batch(a, alg=None, group=None, batch_fn=None):
    """A [B, m, n] float64 / complex128 batch split over the ranks of
    ``group`` (matrices are independent, no collective but the
    gather of the 8- or 16-byte results).  Rank r evaluates its contiguous
    slice with the batch kernels (``alg`` as in ``opt_batch``: None = batch
    dispatch, or "glynn" / "ryser" / "combinatoric"); one all-gather returns
    the whole [B] result on every rank, in batch order.  ``batch_fn`` lets
    tests substitute a CPU evaluator (gloo, no device)."""
    import torch
    import torch.distributed as dist

    from .batch import _run

    arr = np.asarray(a)
    if arr.ndim != 3:
        raise TypeError(f"expected a [B, m, n] array, got ndim={arr.ndim}")
    cplx = np.iscomplexobj(arr)
    rank, world, backend = _world(group)
    B = arr.shape[0]
    b0, b1 = batch_slice(B, rank, world)
    part = arr[b0:b1]
    vals = np.asarray(batch_fn(part) if batch_fn is not None else _run(part, alg),
                      dtype=np.complex128 if cplx else np.float64)
    if world == 1:
        return vals
    # equal-size slots for all_gather_into_tensor: pad every slice to the
    # largest, as real doubles (complex -> 2 doubles per matrix)
    w = 2 if cplx else 1
    slot = -(-B // world)
    buf = np.zeros(slot * w)
    buf[: (b1 - b0) * w] = vals.view(np.float64)
    dev = "cuda" if backend == "nccl" else "cpu"
    t = torch.from_numpy(buf).to(dev)
    gathered = torch.empty(world * slot * w, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(gathered, t, group=group)
    g = gathered.cpu().numpy().reshape(world, slot * w)
    out = np.concatenate([g[r, : (batch_slice(B, r, world)[1] - batch_slice(B, r, world)[0]) * w]
                          for r in range(world)])
    return out.view(np.complex128) if cplx else out
