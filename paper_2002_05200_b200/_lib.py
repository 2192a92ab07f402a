"""ctypes binding of the C ABI in ``include/logan_xdrop.h`` (argument marshalling only).

Every step of the hot path runs in ``liblogan_xdrop.so`` (sm_100a).  There is
no CPU fallback: if the library is missing, or no CUDA device is present, the
calls raise.
"""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "liblogan_xdrop.so")

LOGAN_SEQ_U8 = 0
LOGAN_SEQ_2BIT = 1
LOGAN_OK, LOGAN_EINVAL, LOGAN_ECUDA, LOGAN_ENOSPC = 0, 1, 2, 3
ABI_VERSION = 3  # LOGAN_ABI_VERSION this binding marshals for

#: every symbol include/logan_xdrop.h declares
EXPORTS = ("logan_workspace_bytes", "logan_xdrop_batch", "logan_host_arena_bytes",
           "logan_xdrop_batch_host", "logan_xdrop_batch_host_async", "logan_strerror",
           "logan_abi_version", "logan_level_width", "logan_pack_2bit_bytes", "logan_pack_2bit")


class Scoring(ctypes.Structure):
    _fields_ = [("match", ctypes.c_int32), ("mismatch", ctypes.c_int32),
                ("gap", ctypes.c_int32), ("xdrop", ctypes.c_int32)]


N_STAGES = 10  # LOGAN_N_STAGES: 0 setup, 1..8 levels, 9 combine


class Options(ctypes.Structure):
    _fields_ = [("first_level", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("timing_events", ctypes.c_void_p), ("handover", ctypes.c_int32),
                ("first_slots", ctypes.c_int32), ("subst", ctypes.c_void_p),
                ("alphabet", ctypes.c_int32), ("zdrop", ctypes.c_int32), ("reserved", ctypes.c_int64 * 3)]


class Result(ctypes.Structure):
    _fields_ = [("score", ctypes.c_int32), ("q_begin", ctypes.c_int32), ("q_end", ctypes.c_int32),
                ("t_begin", ctypes.c_int32), ("t_end", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("tasks_started", ctypes.c_uint64 * 8), ("tasks_finished", ctypes.c_uint64 * 8),
                ("cells_per_level", ctypes.c_uint64 * 8), ("window_shifts", ctypes.c_uint64),
                ("cells_total", ctypes.c_uint64), ("pairs_invalid", ctypes.c_uint64),
                ("helper_tasks", ctypes.c_uint64), ("first_level", ctypes.c_uint32),
                ("first_width", ctypes.c_uint32), ("first_shape", ctypes.c_uint32),
                ("first_helpers", ctypes.c_uint32)]


class LoganError(RuntimeError):
    pass


_lib = None


def load(path: str | None = None) -> ctypes.CDLL:
    """Load the library (once).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("LOGAN_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise LoganError(f"{path} is missing: build it with `python -m paper_2002_05200_b200.build` "
                         "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
    lib.logan_workspace_bytes.argtypes = [i64, i64]
    lib.logan_workspace_bytes.restype = sz
    lib.logan_host_arena_bytes.argtypes = [i64, i64, i32, i64]
    lib.logan_host_arena_bytes.restype = sz
    lib.logan_xdrop_batch.argtypes = [vp, i32, i64, vp, vp, vp, vp, vp, vp, i64, i64, i32, Scoring,
                                      ctypes.POINTER(Options), vp, vp, vp, vp, sz, vp]
    lib.logan_xdrop_batch.restype = ctypes.c_int
    lib.logan_xdrop_batch_host.argtypes = [vp, i32, i64, vp, vp, vp, vp, vp, vp, i64, i32, Scoring,
                                           ctypes.POINTER(Options), vp, vp, vp, sz, vp]
    lib.logan_xdrop_batch_host.restype = ctypes.c_int
    lib.logan_xdrop_batch_host_async.argtypes = lib.logan_xdrop_batch_host.argtypes
    lib.logan_xdrop_batch_host_async.restype = ctypes.c_int
    lib.logan_strerror.argtypes = [ctypes.c_int]
    lib.logan_strerror.restype = ctypes.c_char_p
    lib.logan_abi_version.argtypes = []
    lib.logan_abi_version.restype = ctypes.c_int
    lib.logan_level_width.argtypes = [i32, i32, i64, i32]
    lib.logan_level_width.restype = ctypes.c_int
    lib.logan_pack_2bit_bytes.argtypes = [i64]
    lib.logan_pack_2bit_bytes.restype = sz
    lib.logan_pack_2bit.argtypes = [vp, i64, vp, vp, vp, vp, i64, vp, sz, vp, vp]
    lib.logan_pack_2bit.restype = ctypes.c_int
    if lib.logan_abi_version() != ABI_VERSION:
        raise LoganError(f"{path}: ABI version {lib.logan_abi_version()}, binding expects {ABI_VERSION} "
                         "(rebuild with `python -m paper_2002_05200_b200.build`)")
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != LOGAN_OK:
        msg = load().logan_strerror(status).decode()
        raise LoganError(f"logan status {status}: {msg}")
