"""Python API over the C ABI (torch owns device memory and streams).

``xdrop_batch`` takes CUDA tensors and calls ``logan_xdrop_batch`` on the
current torch stream; ``xdrop_batch_host`` takes host numpy arrays (pinned or
not) and calls ``logan_xdrop_batch_host`` (copies in, sweep, copies out) --
the end-to-end entry point.  Nothing here computes any part of the method.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib


def _require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise _lib.LoganError("logan: no CUDA device (this library has no CPU path)")
    return torch


@dataclass
class Workspace:
    """A reusable device workspace (torch uint8 tensor, 256-byte aligned)."""
    tensor: object
    n_pairs: int
    max_ext_len: int

    @property
    def nbytes(self) -> int:
        return int(self.tensor.numel())

    def ptr(self) -> int:
        return int(self.tensor.data_ptr())


def workspace_bytes(n_pairs: int, max_ext_len: int) -> int:
    return int(_lib.load().logan_workspace_bytes(int(n_pairs), int(max_ext_len)))


# One workspace per (device, stream), grown on demand and reused by every call on that
# stream that passes none: stream order makes the reuse safe, and a call does not leave
# a multi-GB block to the caching allocator that it cannot hand out again until the
# stream's kernels finish (record_stream).
_WS_CACHE: dict = {}


def _cached_workspace(n_pairs: int, max_ext_len: int, device, stream) -> Workspace:
    key = (str(device), int(stream.cuda_stream))
    ws = _WS_CACHE.get(key)
    if ws is None or ws.n_pairs < n_pairs or ws.max_ext_len < max_ext_len:
        if ws is not None:
            n_pairs, max_ext_len = max(n_pairs, ws.n_pairs), max(max_ext_len, ws.max_ext_len)
        ws = make_workspace(n_pairs, max_ext_len, device)
        _WS_CACHE[key] = ws
    return ws


def clear_workspace_cache() -> None:
    """Drop the per-stream workspaces ``xdrop_batch`` keeps when it is passed none."""
    _WS_CACHE.clear()


def make_workspace(n_pairs: int, max_ext_len: int, device=None) -> Workspace:
    torch = _require_cuda()
    nb = workspace_bytes(n_pairs, max_ext_len)
    t = torch.empty(max(nb, 256) + 256, dtype=torch.uint8, device=device or "cuda")
    off = (-t.data_ptr()) % 256
    return Workspace(t[off:off + max(nb, 256)], n_pairs, max_ext_len)


def _opts(first_level: int | None, timing_events=None, latency_first: bool = False,
          handover: int = 0, first_slots: int = 0, poison: bool = False, subst=None, zdrop: int | None = None,
          throughput_first: bool = False, nopack: bool = False, compat: bool = False,
          copy_ahead: bool = False):
    """Options struct; ``timing_events`` = list of 2*N_STAGES torch.cuda.Event;
    ``subst`` = square int8 CUDA tensor (alphabet x alphabet) or None."""
    if not first_level and timing_events is None and not latency_first and not handover \
            and not first_slots and not poison and subst is None and zdrop is None and not throughput_first \
            and not nopack and not compat and not copy_ahead:
        return None
    o = _lib.Options()
    o.first_level = int(first_level or 0)
    o.flags = (1 if latency_first else 0) | (2 if poison else 0) | (4 if zdrop is not None else 0) \
        | (8 if throughput_first else 0) | (16 if nopack else 0) | (32 if compat else 0) \
        | (64 if copy_ahead else 0)
    o.zdrop = int(zdrop) if zdrop is not None else 0
    o.handover = int(handover)
    o.first_slots = int(first_slots)
    if subst is not None:
        if subst.dim() != 2 or subst.shape[0] != subst.shape[1] or not subst.is_cuda or \
                not subst.is_contiguous() or str(subst.dtype) != "torch.int8":
            raise ValueError("subst must be a contiguous square int8 CUDA tensor")
        o.subst = subst.data_ptr()
        o.alphabet = int(subst.shape[0])
        o._keep_subst = subst
    if timing_events is not None:
        assert len(timing_events) == 2 * _lib.N_STAGES
        arr = (ctypes.c_void_p * (2 * _lib.N_STAGES))(*[int(e.cuda_event) for e in timing_events])
        o.timing_events = ctypes.cast(arr, ctypes.c_void_p)
        o._keep = arr  # keep the array alive for the call
    return ctypes.pointer(o)


@dataclass
class DeviceBatch:
    """Pairs resident on one device (torch CUDA tensors)."""
    pool: object       # uint8, padded to 16 bytes
    fmt: int
    pool_len: int      # bases
    q_off: object      # int64
    q_len: object      # int32
    t_off: object      # int64
    t_len: object      # int32
    q_seed: object     # int32
    t_seed: object     # int32
    k: int
    max_ext_len: int

    @property
    def n_pairs(self) -> int:
        return int(self.q_len.numel())


def to_device(batch, fmt: int = _lib.LOGAN_SEQ_2BIT, device=None) -> DeviceBatch:
    """Copy a ``datagen.Batch`` (or anything with the same fields) to the GPU."""
    torch = _require_cuda()
    dev = device or "cuda"
    pool = batch.pool_2bit if fmt == _lib.LOGAN_SEQ_2BIT else batch.pool_u8
    if pool is None:
        raise ValueError("batch has no pool in the requested format")
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)
    return DeviceBatch(t(pool, torch.uint8), fmt, int(batch.pool_len),
                       t(batch.q_off, torch.int64), t(batch.q_len, torch.int32),
                       t(batch.t_off, torch.int64), t(batch.t_len, torch.int32),
                       t(batch.q_seed, torch.int32), t(batch.t_seed, torch.int32),
                       int(batch.workload.k), int(batch.max_ext_len()))


def xdrop_batch(db: DeviceBatch, match: int, mismatch: int, gap: int, xdrop: int,
                workspace: Workspace | None = None, out=None, cells=None, stats=None,
                first_level: int | None = None, stream=None, timing_events=None,
                latency_first: bool = False, handover: int = 0, first_slots: int = 0,
                poison: bool = False, subst=None, zdrop: int | None = None, throughput_first: bool = False,
                nopack: bool = False, compat: bool = False, pack_u8: bool = False):
    """Run the whole hot path on ``db``'s device, asynchronously on ``stream``
    (default: torch's current stream).  Returns ``(out int32[n,5], cells int64[n])``
    device tensors (cells holds uint64 bit patterns).

    ``pack_u8=True`` with a ``LOGAN_SEQ_U8`` pool (no ``subst``): re-encode the pool
    as 2-bit on the device first (``logan_pack_2bit``) and run on that copy if every
    base is A/C/G/T -- identical results; this costs one synchronisation of
    ``stream`` (reading the count of other bytes)."""
    torch = _require_cuda()
    lib = _lib.load()
    n = db.n_pairs
    dev = db.q_len.device
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    if pack_u8 and db.fmt == _lib.LOGAN_SEQ_U8 and subst is None and n > 0:
        # the 2-bit copy goes to a buffer kept per (device, stream), like the workspace
        key = ("pack", str(dev), int(stream.cuda_stream))
        nb = int(lib.logan_pack_2bit_bytes(db.pool_len))
        buf = _WS_CACHE.get(key)
        if buf is None or buf[0].numel() < nb:
            buf = (torch.empty(nb, dtype=torch.uint8, device=dev), torch.empty(1, dtype=torch.int64, device=dev))
            _WS_CACHE[key] = buf
        packed, other = pack_2bit(db, stream, into=buf)
        stream.synchronize()
        if int(other.item()) == 0:
            db = packed
    # the library launches on the current device: make it db's (multi-GPU callers)
    with torch.cuda.device(dev):
        if out is None:
            out = torch.empty((n, 5), dtype=torch.int32, device=dev)
        if cells is None:
            cells = torch.empty(n, dtype=torch.int64, device=dev)
        if workspace is None:
            workspace = _cached_workspace(n, db.max_ext_len, dev, stream)
        elif workspace.n_pairs < n or workspace.max_ext_len < db.max_ext_len:
            workspace = make_workspace(n, db.max_ext_len, dev)
        # the kernels run asynchronously on `stream`: keep the caching allocator from
        # handing these blocks to another stream's allocation before they finish
        for t in (out, cells, workspace.tensor):
            t.record_stream(stream)
        sc = _lib.Scoring(match, mismatch, gap, xdrop)
        st = lib.logan_xdrop_batch(
            db.pool.data_ptr(), db.fmt, db.pool_len, db.q_off.data_ptr(), db.q_len.data_ptr(),
            db.t_off.data_ptr(), db.t_len.data_ptr(), db.q_seed.data_ptr(), db.t_seed.data_ptr(),
            n, db.max_ext_len, db.k, sc,
            _opts(first_level, timing_events, latency_first, handover, first_slots, poison, subst, zdrop,
                  throughput_first, nopack, compat),
            out.data_ptr(),
            cells.data_ptr(),
            stats.data_ptr() if stats is not None else None,
            workspace.ptr(), workspace.nbytes, stream.cuda_stream)
    _lib.check(st)
    return out, cells


def pack_2bit(db: DeviceBatch, stream=None, into=None):
    """``logan_pack_2bit``: a 2-bit copy of ``db``'s u8 pool (same descriptors) and a
    device int64 tensor with the number of bytes outside A/C/G/T inside ``db``'s reads
    (the copy is equivalent only if it is 0), both on ``stream``; no synchronisation.
    ``into`` = (uint8 tensor, int64 tensor) to write instead of fresh allocations."""
    torch = _require_cuda()
    lib = _lib.load()
    if db.fmt != _lib.LOGAN_SEQ_U8:
        raise ValueError("pack_2bit needs a LOGAN_SEQ_U8 pool")
    dev = db.pool.device
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    nb = int(lib.logan_pack_2bit_bytes(db.pool_len))
    with torch.cuda.device(dev):
        if into is not None and into[0].numel() >= nb:
            pool, other = into
        else:
            pool = torch.empty(nb, dtype=torch.uint8, device=dev)
            other = torch.empty(1, dtype=torch.int64, device=dev)
        for t in (pool, other):
            t.record_stream(stream)
        _lib.check(lib.logan_pack_2bit(db.pool.data_ptr(), db.pool_len, db.q_off.data_ptr(), db.q_len.data_ptr(),
                                       db.t_off.data_ptr(), db.t_len.data_ptr(), db.n_pairs, pool.data_ptr(), nb,
                                       other.data_ptr(), stream.cuda_stream))
    return DeviceBatch(pool, _lib.LOGAN_SEQ_2BIT, db.pool_len, db.q_off, db.q_len, db.t_off, db.t_len,
                       db.q_seed, db.t_seed, db.k, db.max_ext_len), other


def new_stats(device=None):
    torch = _require_cuda()
    return torch.zeros(ctypes.sizeof(_lib.Stats) // 8, dtype=torch.int64, device=device or "cuda")


def stats_dict(stats_tensor) -> dict:
    v = [int(x) for x in stats_tensor.cpu().tolist()]
    return {"tasks_started": v[0:8], "tasks_finished": v[8:16], "cells_per_level": v[16:24],
            "window_shifts": v[24], "cells_total": v[25], "pairs_invalid": v[26], "helper_tasks": v[27],
            "first_level": v[28] & 0xffffffff, "first_width": v[28] >> 32,
            "first_shape": "latency" if v[29] & 0xffffffff else "throughput", "first_helpers": bool(v[29] >> 32)}


class HostArena:
    """Device arena for the host-buffer entry point (allocated once, reused)."""

    def __init__(self, n_pairs: int, pool_len: int, fmt: int, max_ext_len: int, device=None):
        torch = _require_cuda()
        nb = int(_lib.load().logan_host_arena_bytes(n_pairs, pool_len, fmt, max_ext_len))
        t = torch.empty(nb + 256, dtype=torch.uint8, device=device or "cuda")
        off = (-t.data_ptr()) % 256
        self.tensor = t[off:off + nb]
        self.nbytes = nb


def xdrop_batch_host(pool: np.ndarray, fmt: int, pool_len: int, q_off, q_len, t_off, t_len,
                     q_seed, t_seed, k: int, match: int, mismatch: int, gap: int, xdrop: int,
                     arena: HostArena, out: np.ndarray | None = None,
                     cells: np.ndarray | None = None, first_level: int | None = None, stream=None,
                     asynchronous: bool = False, subst=None, zdrop: int | None = None,
                     copy_ahead: bool = False, timing_events=None):
    """End-to-end call with HOST buffers (numpy; pinned memory copies fastest).

    ``asynchronous=True`` returns right after enqueuing (``logan_xdrop_batch_host_async``):
    the outputs are valid once ``stream`` is synchronised and the inputs must stay alive
    until then. ``copy_ahead=True`` (asynchronous calls; options.flags bit 6) copies the
    inputs on a library stream as soon as ``arena`` is free instead of when ``stream``
    reaches the call: with one stream and a ring of arenas, every step's copies overlap
    the previous sweeps."""
    torch = _require_cuda()
    lib = _lib.load()
    n = len(q_len)
    if out is None:
        out = np.empty((n, 5), np.int32)
    if cells is None:
        cells = np.empty(n, np.uint64)
    arrs = [np.ascontiguousarray(a) for a in (q_off, q_len, t_off, t_len, q_seed, t_seed)]
    if asynchronous and any(a is not b for a, b in zip(arrs, (q_off, q_len, t_off, t_len, q_seed, t_seed))):
        raise ValueError("asynchronous host calls need C-contiguous numpy inputs (they must outlive the call)")
    dev = arena.tensor.device
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    sc = _lib.Scoring(match, mismatch, gap, xdrop)
    ptr = lambda a: a.ctypes.data
    fn = lib.logan_xdrop_batch_host_async if asynchronous else lib.logan_xdrop_batch_host
    with torch.cuda.device(dev):
        st = fn(ptr(pool), fmt, pool_len, *[ptr(a) for a in arrs], n, k, sc,
                _opts(first_level, timing_events, subst=subst, zdrop=zdrop, copy_ahead=copy_ahead), ptr(out), ptr(cells),
                arena.tensor.data_ptr(), arena.nbytes, stream.cuda_stream)
    _lib.check(st)
    return out, cells
