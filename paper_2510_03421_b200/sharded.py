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


def sharded_permanent(a, alg: str = "glynn", group=None, mag: bool = False, partial_fn=None):
    """Permanent of one m x n (m <= n) float64 / complex128 matrix with its
    walk sharded over the ranks of ``group`` (default: the world).  Every
    rank returns the same value.  Returns (value, M) if ``mag`` else value."""
    import torch
    import torch.distributed as dist

    a = np.asarray(a)
    if a.shape[0] > a.shape[1]:
        a = a.T
    a = np.ascontiguousarray(a, dtype=np.complex128 if np.iscomplexobj(a) else np.float64)
    m, n = a.shape
    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        backend = dist.get_backend(group)
    else:
        rank, world, backend = 0, 1, None
    k0, k1 = shard_range(alg, m, n, rank, world)
    if partial_fn is not None:
        part = torch.tensor(np.asarray(partial_fn(alg, a, k0, k1), dtype=np.float64))
    elif backend == "nccl":
        part = torch.empty(8, dtype=torch.float64, device="cuda")
        gpu_partial(alg, a, k0, k1, mag, device_out=part, stream=torch.cuda.current_stream().cuda_stream)
    else:
        part = torch.tensor(gpu_partial(alg, a, k0, k1, mag))
    if world > 1:
        gathered = torch.empty(world * 8, dtype=torch.float64, device=part.device)
        dist.all_gather_into_tensor(gathered, part, group=group)
        parts = gathered.cpu().numpy()
    else:
        parts = part.cpu().numpy()
    value, M = finish(alg, a, parts)
    return (value, M) if mag else value
