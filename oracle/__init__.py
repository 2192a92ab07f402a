"""CPU oracle for LOGAN's batched X-drop seed-and-extend (arXiv 2002.05200).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import
this package.  The product path (``paper_2002_05200_b200``) never imports it
and shares no code with it; the two meet only in the tests, which feed both
the same seeded inputs from ``datagen``.

Contents
--------
* ``xdrop_oracle.c`` (compiled to ``_liboracle.so`` by :func:`build`): the
  plain C oracle -- definition, citations and readings in its header.
* :func:`extend`, :func:`pair`, :func:`pairs`: ctypes bindings.
* :mod:`oracle.tiny`: a pure-Python dict-of-live-cells oracle and a
  brute-force full-matrix DP, for the pins on tiny inputs.

Parity status: every function is pinned by the tests in
``tests/test_oracle_pins.py`` (closed forms, X = inf brute force, hand-worked
examples under ``tests/golden/``, invariants).  The paper prints no per-pair
value, so no pin is a value printed by the paper.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "xdrop_oracle.c")
_LIB = os.path.join(_HERE, "_liboracle.so")


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (plain -O2, no vectorisation flags)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-o", tmp, _SRC]
        )
        os.replace(tmp, _LIB)
    return _LIB


class _Ext(ctypes.Structure):
    _fields_ = [("best", ctypes.c_int64), ("i", ctypes.c_int64), ("j", ctypes.c_int64),
                ("cells", ctypes.c_uint64), ("last_d", ctypes.c_int64)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i64, i32p, i64p = ctypes.c_int64, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        lib.oracle_extend.argtypes = [u8p, i64, u8p, i64, i64, i64, i64, i64, ctypes.c_int,
                                      ctypes.POINTER(_Ext)]
        lib.oracle_extend.restype = ctypes.c_int
        lib.oracle_pairs.argtypes = [u8p, ctypes.c_int, i64, i64p, i32p, i64p, i32p, i32p, i32p,
                                     i64, i64, i64, i64, i64, i64, i32p,
                                     ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
        lib.oracle_pairs.restype = ctypes.c_int
        i8p = ctypes.POINTER(ctypes.c_int8)
        lib.oracle_extend_subst.argtypes = [u8p, i64, u8p, i64, i8p, i64, i64, i64, ctypes.c_int,
                                            ctypes.POINTER(_Ext)]
        lib.oracle_extend_subst.restype = ctypes.c_int
        lib.oracle_pairs_subst.argtypes = [u8p, i64, i64p, i32p, i64p, i32p, i32p, i32p,
                                           i64, i64, i8p, i64, i64, i64, i32p,
                                           ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
        lib.oracle_pairs_subst.restype = ctypes.c_int
        lib.oracle_extend_z.argtypes = [u8p, i64, u8p, i64, i64, i64, i8p, i64, i64, i64, i64, ctypes.c_int,
                                        ctypes.POINTER(_Ext)]
        lib.oracle_extend_z.restype = ctypes.c_int
        lib.oracle_pairs_z.argtypes = [u8p, ctypes.c_int, i64, i64p, i32p, i64p, i32p, i32p, i32p,
                                       i64, i64, i64, i64, i8p, i64, i64, i64, i64, i32p,
                                       ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
        lib.oracle_pairs_z.restype = ctypes.c_int
        lib.oracle_extend_compat.argtypes = [u8p, i64, u8p, i64, i64, i64, i64, i64, i64, ctypes.c_int,
                                             ctypes.POINTER(_Ext)]
        lib.oracle_extend_compat.restype = ctypes.c_int
        lib.oracle_pairs_compat.argtypes = [u8p, ctypes.c_int, i64, i64p, i32p, i64p, i32p, i32p, i32p,
                                            i64, i64, i64, i64, i64, i64, i64, i32p,
                                            ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
        lib.oracle_pairs_compat.restype = ctypes.c_int
        _lib = lib
    return _lib


@dataclass(frozen=True)
class ExtResult:
    best: int
    i: int
    j: int
    cells: int
    last_d: int


def _as_u8(s) -> np.ndarray:
    if isinstance(s, str):
        s = s.encode()
    return np.frombuffer(bytes(s), dtype=np.uint8) if not isinstance(s, np.ndarray) else \
        np.ascontiguousarray(s, dtype=np.uint8)


def extend(A, B, X: int, match: int = 1, mismatch: int = -1, gap: int = -1,
           full_scan: bool = False) -> ExtResult:
    """One X-drop extension E(A, B) (oracle header steps 1-5)."""
    a, b = _as_u8(A), _as_u8(B)
    out = _Ext()
    u8p = ctypes.POINTER(ctypes.c_uint8)
    st = _load().oracle_extend(a.ctypes.data_as(u8p), len(a), b.ctypes.data_as(u8p), len(b),
                               match, mismatch, gap, X, int(full_scan), ctypes.byref(out))
    if st != 0:
        raise RuntimeError(f"oracle_extend failed with status {st}")
    return ExtResult(out.best, out.i, out.j, out.cells, out.last_d)


def pairs(pool: np.ndarray, fmt: int, q_off, q_len, t_off, t_len, q_seed, t_seed, k: int,
          match: int, mismatch: int, gap: int, X: int, pool_len: int | None = None,
          n_threads: int | None = None):
    """Batch of pairs -> (int32[n,5] results, uint64[n] cells).

    ``fmt`` 0 = u8 pool, 1 = 2-bit pool; ``pool_len`` in bases (defaults to the
    whole buffer).  Runs ``n_threads`` host threads (default: all cores this
    process may use), each executing the single-threaded oracle pair by pair.
    """
    pool = np.ascontiguousarray(pool, dtype=np.uint8)
    if pool_len is None:
        pool_len = len(pool) if fmt == 0 else 4 * len(pool)
    cols = [np.ascontiguousarray(x, dtype=dt) for x, dt in
            ((q_off, np.int64), (q_len, np.int32), (t_off, np.int64), (t_len, np.int32),
             (q_seed, np.int32), (t_seed, np.int32))]
    n = len(cols[0])
    out = np.zeros((n, 5), dtype=np.int32)
    cells = np.zeros(n, dtype=np.uint64)
    if n_threads is None:
        n_threads = len(os.sched_getaffinity(0))
    P = ctypes.POINTER
    st = _load().oracle_pairs(
        pool.ctypes.data_as(P(ctypes.c_uint8)), fmt, pool_len,
        cols[0].ctypes.data_as(P(ctypes.c_int64)), cols[1].ctypes.data_as(P(ctypes.c_int32)),
        cols[2].ctypes.data_as(P(ctypes.c_int64)), cols[3].ctypes.data_as(P(ctypes.c_int32)),
        cols[4].ctypes.data_as(P(ctypes.c_int32)), cols[5].ctypes.data_as(P(ctypes.c_int32)),
        n, k, match, mismatch, gap, X,
        out.ctypes.data_as(P(ctypes.c_int32)), cells.ctypes.data_as(P(ctypes.c_uint64)),
        int(n_threads))
    if st != 0:
        raise RuntimeError(f"oracle_pairs failed with status {st}")
    return out, cells


def pair(q, t, qs: int, ts: int, k: int, X: int, match: int = 1, mismatch: int = -1,
         gap: int = -1):
    """One pair given as two byte strings -> ((score, qb, qe, tb, te), cells)."""
    qa, ta = _as_u8(q), _as_u8(t)
    pool = np.concatenate([qa, ta])
    out, cells = pairs(pool, 0, [0], [len(qa)], [len(qa)], [len(ta)], [qs], [ts], k,
                       match, mismatch, gap, X, n_threads=1)
    return tuple(int(x) for x in out[0]), int(cells[0])


def _subst_table(subst) -> tuple[np.ndarray, int]:
    t = np.ascontiguousarray(subst, dtype=np.int8)
    if t.ndim != 2 or t.shape[0] != t.shape[1]:
        raise ValueError("subst must be a square alphabet x alphabet matrix")
    return t, t.shape[0]


def extend_subst(A, B, X: int, subst, gap: int, full_scan: bool = False) -> ExtResult:
    """One X-drop extension scored with a substitution matrix:
    s(a_i, b_j) = subst[a_i][b_j] (codes 0..alphabet-1)."""
    a, b = _as_u8(A), _as_u8(B)
    t, alph = _subst_table(subst)
    out = _Ext()
    P = ctypes.POINTER
    st = _load().oracle_extend_subst(a.ctypes.data_as(P(ctypes.c_uint8)), len(a),
                                     b.ctypes.data_as(P(ctypes.c_uint8)), len(b),
                                     t.ctypes.data_as(P(ctypes.c_int8)), alph, gap, X, int(full_scan),
                                     ctypes.byref(out))
    if st != 0:
        raise RuntimeError(f"oracle_extend_subst failed with status {st}")
    return ExtResult(out.best, out.i, out.j, out.cells, out.last_d)


def pairs_subst(pool: np.ndarray, q_off, q_len, t_off, t_len, q_seed, t_seed, k: int, subst,
                gap: int, X: int, pool_len: int | None = None, n_threads: int | None = None):
    """Batch of pairs in a u8 pool of codes < alphabet, scored with ``subst``
    -> (int32[n,5] results, uint64[n] cells)."""
    pool = np.ascontiguousarray(pool, dtype=np.uint8)
    t, alph = _subst_table(subst)
    if pool_len is None:
        pool_len = len(pool)
    cols = [np.ascontiguousarray(x, dtype=dt) for x, dt in
            ((q_off, np.int64), (q_len, np.int32), (t_off, np.int64), (t_len, np.int32),
             (q_seed, np.int32), (t_seed, np.int32))]
    n = len(cols[0])
    out = np.zeros((n, 5), dtype=np.int32)
    cells = np.zeros(n, dtype=np.uint64)
    if n_threads is None:
        n_threads = len(os.sched_getaffinity(0))
    P = ctypes.POINTER
    st = _load().oracle_pairs_subst(
        pool.ctypes.data_as(P(ctypes.c_uint8)), pool_len,
        cols[0].ctypes.data_as(P(ctypes.c_int64)), cols[1].ctypes.data_as(P(ctypes.c_int32)),
        cols[2].ctypes.data_as(P(ctypes.c_int64)), cols[3].ctypes.data_as(P(ctypes.c_int32)),
        cols[4].ctypes.data_as(P(ctypes.c_int32)), cols[5].ctypes.data_as(P(ctypes.c_int32)),
        n, k, t.ctypes.data_as(P(ctypes.c_int8)), alph, gap, X,
        out.ctypes.data_as(P(ctypes.c_int32)), cells.ctypes.data_as(P(ctypes.c_uint64)),
        int(n_threads))
    if st != 0:
        raise RuntimeError(f"oracle_pairs_subst failed with status {st}")
    return out, cells


def extend_z(A, B, X: int, zdrop: int, match: int = 1, mismatch: int = -1, gap: int = -1, subst=None,
             full_scan: bool = False) -> ExtResult:
    """X-drop extension with the optional Z-drop stop (oracle header step 3b;
    ``zdrop`` < 0 = off) and optional substitution matrix."""
    a, b = _as_u8(A), _as_u8(B)
    P = ctypes.POINTER
    t, alph = (_subst_table(subst) if subst is not None else (None, 0))
    tp = t.ctypes.data_as(P(ctypes.c_int8)) if t is not None else None
    out = _Ext()
    st = _load().oracle_extend_z(a.ctypes.data_as(P(ctypes.c_uint8)), len(a), b.ctypes.data_as(P(ctypes.c_uint8)),
                                 len(b), match, mismatch, tp, alph, gap, X, zdrop, int(full_scan), ctypes.byref(out))
    if st != 0:
        raise RuntimeError(f"oracle_extend_z failed with status {st}")
    return ExtResult(out.best, out.i, out.j, out.cells, out.last_d)


def pairs_z(pool: np.ndarray, fmt: int, q_off, q_len, t_off, t_len, q_seed, t_seed, k: int, match: int,
            mismatch: int, gap: int, X: int, zdrop: int, subst=None, pool_len: int | None = None,
            n_threads: int | None = None):
    """Batch with Z-drop (``zdrop`` < 0 = off) and an optional substitution
    matrix (then ``fmt`` must be 0, a u8 pool of codes)."""
    pool = np.ascontiguousarray(pool, dtype=np.uint8)
    if pool_len is None:
        pool_len = len(pool) if fmt == 0 else 4 * len(pool)
    t, alph = (_subst_table(subst) if subst is not None else (None, 0))
    cols = [np.ascontiguousarray(x, dtype=dt) for x, dt in
            ((q_off, np.int64), (q_len, np.int32), (t_off, np.int64), (t_len, np.int32),
             (q_seed, np.int32), (t_seed, np.int32))]
    n = len(cols[0])
    out = np.zeros((n, 5), dtype=np.int32)
    cells = np.zeros(n, dtype=np.uint64)
    if n_threads is None:
        n_threads = len(os.sched_getaffinity(0))
    P = ctypes.POINTER
    st = _load().oracle_pairs_z(
        pool.ctypes.data_as(P(ctypes.c_uint8)), fmt, pool_len,
        cols[0].ctypes.data_as(P(ctypes.c_int64)), cols[1].ctypes.data_as(P(ctypes.c_int32)),
        cols[2].ctypes.data_as(P(ctypes.c_int64)), cols[3].ctypes.data_as(P(ctypes.c_int32)),
        cols[4].ctypes.data_as(P(ctypes.c_int32)), cols[5].ctypes.data_as(P(ctypes.c_int32)),
        n, k, match, mismatch, t.ctypes.data_as(P(ctypes.c_int8)) if t is not None else None, alph, gap, X,
        zdrop, out.ctypes.data_as(P(ctypes.c_int32)), cells.ctypes.data_as(P(ctypes.c_uint64)), int(n_threads))
    if st != 0:
        raise RuntimeError(f"oracle_pairs_z failed with status {st}")
    return out, cells


def extend_compat(A, B, X: int, match: int = 1, mismatch: int = -1, gap: int = -1, zdrop: int = -1,
                  full_scan: bool = False) -> ExtResult:
    """SeqAn-compat extension (oracle header step 6; [outside-PAPER] readings
    c-amb-24/25): strict boundary drop for d >= 2, (i, j) = the longest-extension
    cell (the best live cell of the last live antidiagonal)."""
    a, b = _as_u8(A), _as_u8(B)
    out = _Ext()
    u8p = ctypes.POINTER(ctypes.c_uint8)
    st = _load().oracle_extend_compat(a.ctypes.data_as(u8p), len(a), b.ctypes.data_as(u8p), len(b),
                                      match, mismatch, gap, X, zdrop, int(full_scan), ctypes.byref(out))
    if st != 0:
        raise RuntimeError(f"oracle_extend_compat failed with status {st}")
    return ExtResult(out.best, out.i, out.j, out.cells, out.last_d)


def pairs_compat(pool: np.ndarray, fmt: int, q_off, q_len, t_off, t_len, q_seed, t_seed, k: int,
                 match: int, mismatch: int, gap: int, X: int, zdrop: int = -1, pool_len: int | None = None,
                 n_threads: int | None = None):
    """Batch of pairs in SeqAn-compat mode -> (int32[n,5], uint64[n])."""
    pool = np.ascontiguousarray(pool, dtype=np.uint8)
    if pool_len is None:
        pool_len = len(pool) if fmt == 0 else 4 * len(pool)
    cols = [np.ascontiguousarray(x, dtype=dt) for x, dt in
            ((q_off, np.int64), (q_len, np.int32), (t_off, np.int64), (t_len, np.int32),
             (q_seed, np.int32), (t_seed, np.int32))]
    n = len(cols[0])
    out = np.zeros((n, 5), dtype=np.int32)
    cells = np.zeros(n, dtype=np.uint64)
    if n_threads is None:
        n_threads = len(os.sched_getaffinity(0))
    P = ctypes.POINTER
    st = _load().oracle_pairs_compat(
        pool.ctypes.data_as(P(ctypes.c_uint8)), fmt, pool_len,
        cols[0].ctypes.data_as(P(ctypes.c_int64)), cols[1].ctypes.data_as(P(ctypes.c_int32)),
        cols[2].ctypes.data_as(P(ctypes.c_int64)), cols[3].ctypes.data_as(P(ctypes.c_int32)),
        cols[4].ctypes.data_as(P(ctypes.c_int32)), cols[5].ctypes.data_as(P(ctypes.c_int32)),
        n, k, match, mismatch, gap, X, zdrop, out.ctypes.data_as(P(ctypes.c_int32)),
        cells.ctypes.data_as(P(ctypes.c_uint64)), int(n_threads))
    if st != 0:
        raise RuntimeError(f"oracle_pairs_compat failed with status {st}")
    return out, cells
