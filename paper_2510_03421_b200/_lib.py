"""ctypes binding of libpermanent_b200.so (the C ABI in include/permanent_b200.h).

There is no CPU fallback: if the library is missing, or no CUDA device is
visible, every compute call raises ``EngineUnavailable``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libpermanent_b200.so"

OK, OVERFLOW, BAD_SHAPE, BUDGET, CUDA, BAD_ARG = range(6)
ALG_COMBINATORIC, ALG_RYSER, ALG_GLYNN = 0, 1, 2

_lock = threading.Lock()
_lib = None

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int64)
_vp = C.c_void_p

# name -> (restype, argtypes); every symbol include/permanent_b200.h declares
SIGNATURES = {
    "perm_version": (C.c_int, []),
    "perm_last_error": (C.c_char_p, []),
    "perm_set_device": (C.c_int, [C.c_int]),
    "perm_device_sm_count": (C.c_int, []),
    "perm_last_kernel_ms": (C.c_double, []),
    "perm_set_timing": (C.c_int, [C.c_int]),
    "perm_last_kernel_plan": (C.c_int, [C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "perm_fp64_peak_probe": (C.c_int, [C.c_double, _dp]),
    "perm_fp64_pipe_probe": (C.c_int, [C.c_int, C.c_double, _dp]),
    "perm_walk_repeat_ms": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _vp, C.c_int64, C.c_int, _dp]),
    "perm_glynn_f64": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int64, C.c_int, _dp, _dp, _vp]),
    "perm_glynn_c128": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int64, C.c_int, _dp, _dp, _vp]),
    "perm_ryser_f64": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int64, C.c_int, _dp, _dp, _vp]),
    "perm_ryser_c128": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int64, C.c_int, _dp, _dp, _vp]),
    "perm_ryser_rect_f64": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int64, C.c_int, _dp, _vp]),
    "perm_ryser_rect_c128": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int64, C.c_int, _dp, _vp]),
    "perm_ryser_rect_i64": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int64, C.c_int, _ip, _vp]),
    "perm_comb_f64": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int64, C.c_int, C.c_uint64, _dp, _vp]),
    "perm_comb_c128": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int64, C.c_int, C.c_uint64, _dp, _vp]),
    "perm_comb_i64": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int64, C.c_int, C.c_int, C.c_uint64, _ip,
                                C.POINTER(C.c_int), _vp]),
    "perm_glynn_i64": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int64, C.c_int, C.c_int, _ip,
                                 C.POINTER(C.c_int), _vp]),
    "perm_ryser_i64": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int64, C.c_int, C.c_int, _ip,
                                 C.POINTER(C.c_int), _vp]),
    "perm_batch_f64": (C.c_int, [C.c_int, C.c_int64, C.c_int, C.c_int, _vp, _vp, C.c_int, _vp]),
    "perm_batch_c128": (C.c_int, [C.c_int, C.c_int64, C.c_int, C.c_int, _vp, _vp, C.c_int, _vp]),
    "perm_batch_select": (C.c_int, [C.c_int, C.c_int]),
    "perm_permanent_dd": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _vp, C.c_int64, C.c_int, _dp, _vp]),
    "perm_walk_steps": (C.c_uint64, [C.c_int, C.c_int, C.c_int]),
    "perm_walk_shard": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "perm_walk_partial_f64": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.c_int64, C.c_int, C.c_uint64,
                                        C.c_uint64, C.c_int, _vp, C.c_int, _vp]),
    "perm_walk_partial_c128": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.c_int64, C.c_int, C.c_uint64,
                                         C.c_uint64, C.c_int, _vp, C.c_int, _vp]),
    "perm_walk_finish_f64": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.c_int64, _vp, C.c_int, _dp, _dp]),
    "perm_walk_finish_c128": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.c_int64, _vp, C.c_int, _dp, _dp]),
    "perm_int_walk_plan": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.c_int64, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "perm_walk_partial_i64": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.c_int64, C.c_int, C.c_int, C.c_uint64,
                                        C.c_uint64, _ip, _vp]),
    "perm_walk_finish_i64": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.c_int64, C.c_int, _ip, C.c_int, _ip,
                                       C.POINTER(C.c_int)]),
    "perm_sharded_f64": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.c_int64, C.c_int, C.POINTER(C.c_int), _dp,
                                   _dp]),
    "perm_sharded_c128": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.c_int64, C.c_int, C.POINTER(C.c_int), _dp,
                                    _dp]),
    "perm_sharded_i64": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.c_int64, C.c_int, C.c_int,
                                   C.POINTER(C.c_int), _ip, C.POINTER(C.c_int)]),
    "perm_sharded_exchange": (C.c_int, [C.c_int, C.POINTER(C.c_int)]),
    "perm_select": (C.c_int, [C.c_int, C.c_int, _dp, C.c_int64, C.c_int]),
}


class EngineUnavailable(RuntimeError):
    """The CUDA engine library or a CUDA device is missing (no CPU fallback)."""


class EngineError(RuntimeError):
    """A CUDA-side failure reported by the engine."""


def load():
    """Load (once) and return the engine library; raises EngineUnavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("PERMANENT_B200_LIB", str(LIB_PATH))
            if not Path(path).exists():
                raise EngineUnavailable(
                    f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().perm_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str):
    """Map an engine status to the reference's exception types."""
    if status == OK:
        return
    msg = last_error()
    if status == BAD_SHAPE or status == BAD_ARG:
        raise ValueError(f"{what}: {msg}")
    if status == CUDA:
        if "no CUDA-capable device" in msg or "cudaErrorNoDevice" in msg or "no CUDA device" in msg:
            raise EngineUnavailable(f"{what}: {msg}")
        raise EngineError(f"{what}: {msg}")
    raise EngineError(f"{what}: status {status}: {msg}")


def ptr(arr: np.ndarray):
    return C.c_void_p(arr.ctypes.data)


def out_buf(n: int):
    return (C.c_double * n)()
