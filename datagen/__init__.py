"""Seeded synthetic workloads for the LOGAN X-drop hot path.

This module is shared by the oracle tests and the CUDA path and holds none of
the method's arithmetic (no scoring, no DP): it only produces reads, seeds and
the per-workload constants (scoring scheme and X are *inputs* of the method).

Pair ``p`` of a workload is a pure function of ``(seed, p)`` (counter-based
RNG in ``gen.c``), so shards generated on different ranks are slices of the
same global batch.  Recipe: DESIGN.md §5 and the header of ``gen.c``.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field, replace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "_libgen.so")

#: base seed: the arXiv id; config c uses SEED_BASE + c.
SEED_BASE = 2002052000


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-o",
                               tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Cfg(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("n_pairs", ctypes.c_int64),
                ("pair_base", ctypes.c_int64), ("mode", ctypes.c_int32),
                ("tlen_min", ctypes.c_int32), ("tlen_max", ctypes.c_int32),
                ("err", ctypes.c_double), ("k", ctypes.c_int32), ("spurious", ctypes.c_double),
                ("len_lo", ctypes.c_int32), ("len_hi", ctypes.c_int32), ("burst", ctypes.c_double)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        lib.gen_lengths.argtypes = [P(_Cfg)] + [P(ctypes.c_int32)] * 4 + [ctypes.c_int]
        lib.gen_lengths.restype = ctypes.c_int
        lib.gen_bases.argtypes = [P(_Cfg), P(ctypes.c_int64), P(ctypes.c_uint8),
                                  P(ctypes.c_uint8), ctypes.c_int]
        lib.gen_bases.restype = ctypes.c_int
        lib.gen_lengths_idx.argtypes = [P(_Cfg), P(ctypes.c_int64)] + [P(ctypes.c_int32)] * 4 + [ctypes.c_int]
        lib.gen_lengths_idx.restype = ctypes.c_int
        lib.gen_bases_idx.argtypes = [P(_Cfg), P(ctypes.c_int64), P(ctypes.c_int64), P(ctypes.c_uint8),
                                      P(ctypes.c_uint8), ctypes.c_int]
        lib.gen_bases_idx.restype = ctypes.c_int
        _lib = lib
    return _lib


@dataclass(frozen=True)
class Workload:
    """A workload recipe (one of BASELINE.json's configs, or a variant)."""
    name: str
    n_pairs: int
    mode: int = 0            # 0 template pairs, 1 BELLA-like
    tlen_min: int = 1000
    tlen_max: int = 1000
    err: float = 0.15
    k: int = 17
    spurious: float = 0.0
    len_lo: int = 1000
    len_hi: int = 30000
    burst: float = 0.0
    # method inputs (not generator arithmetic): scoring scheme and X
    match: int = 1
    mismatch: int = -1
    gap: int = -1
    xdrop: int = 50
    seed: int = SEED_BASE

    def with_(self, **kw) -> "Workload":
        return replace(self, **kw)

    @property
    def max_read_len(self) -> int:
        # a read is at most twice its template (one insertion per base) plus a burst block
        base = self.len_hi if self.mode == 1 else self.tlen_max
        return 2 * base + 320


#: BASELINE.json configs.  C3 is listed at X = 20; the sweep
#: varies ``xdrop``.  C4 is ~1M pairs at full size.
CONFIGS = {
    1: Workload("c1_1k_x50", 1_000, tlen_min=1000, tlen_max=1000, err=0.15, xdrop=50,
                seed=SEED_BASE + 1),
    2: Workload("c2_2.5k_x20", 100_000, tlen_min=2500, tlen_max=2500, err=0.15, xdrop=20,
                seed=SEED_BASE + 2),
    3: Workload("c3_10k_x20", 100_000, tlen_min=10000, tlen_max=10000, err=0.15, xdrop=20,
                seed=SEED_BASE + 3),
    4: Workload("c4_bella_x50", 1_000_000, mode=1, err=0.15, spurious=0.30, len_lo=1000,
                len_hi=30000, xdrop=50, seed=SEED_BASE + 4),
    5: Workload("c5_long_x100", 20_000, tlen_min=50000, tlen_max=100000, err=0.12, xdrop=100,
                seed=SEED_BASE + 5),
    # not a BASELINE config: the paper's own benchmark set (Tables II-III):
    # 100K pairs of 2.5-7.5 kb reads at ~15% error, swept over X = 10 ... 5000
    # (the wide-band mode); listed at its largest X
    6: Workload("t2_2.5-7.5k_x5000", 100_000, tlen_min=2500, tlen_max=7500, err=0.15, xdrop=5000,
                seed=SEED_BASE + 6),
}


@dataclass
class Batch:
    """Generated pairs.  Offsets/lengths in bases; pools in both formats on request."""
    workload: Workload
    pair_base: int
    q_off: np.ndarray
    q_len: np.ndarray
    t_off: np.ndarray
    t_len: np.ndarray
    q_seed: np.ndarray
    t_seed: np.ndarray
    pool_len: int
    pool_u8: np.ndarray | None = None
    pool_2bit: np.ndarray | None = None
    meta: dict = field(default_factory=dict)

    @property
    def n_pairs(self) -> int:
        return len(self.q_len)

    def max_ext_len(self) -> int:
        if self.n_pairs == 0:
            return 0
        k = self.workload.k
        return int(max(self.q_seed.max(), self.t_seed.max(),
                       (self.q_len - self.q_seed - k).max(), (self.t_len - self.t_seed - k).max(), 0))


def _pad16(n: int) -> int:
    return (n + 15) // 16 * 16


def generate(w: Workload, n_pairs: int | None = None, pair_base: int = 0, u8: bool = True,
             two_bit: bool = True, n_threads: int | None = None, indices=None) -> Batch:
    """Generate pairs ``[pair_base, pair_base + n_pairs)`` of workload ``w``, or
    the global pairs ``indices`` (any order; a shard of a partitioned batch).

    The pools are padded with zero bytes to a multiple of 16 bytes + 16 (the
    library reads whole words).
    """
    idx = None if indices is None else np.ascontiguousarray(indices, np.int64)
    n = (w.n_pairs if n_pairs is None else int(n_pairs)) if idx is None else len(idx)
    if n_threads is None:
        n_threads = len(os.sched_getaffinity(0))
    cfg = _Cfg(w.seed, n, pair_base, w.mode, w.tlen_min, w.tlen_max, w.err, w.k, w.spurious,
               w.len_lo, w.len_hi, w.burst)
    P = ctypes.POINTER
    ql = np.zeros(n, np.int32); tl = np.zeros(n, np.int32)
    qs = np.zeros(n, np.int32); ts = np.zeros(n, np.int32)
    lib = _load()
    ip = idx.ctypes.data_as(P(ctypes.c_int64)) if idx is not None else None
    if n > 0:
        lens = [a.ctypes.data_as(P(ctypes.c_int32)) for a in (ql, tl, qs, ts)]
        st = (lib.gen_lengths(ctypes.byref(cfg), *lens, n_threads) if idx is None else
              lib.gen_lengths_idx(ctypes.byref(cfg), ip, *lens, n_threads))
        if st != 0:
            raise RuntimeError("gen_lengths failed")
    region = (ql.astype(np.int64) + tl + 3) // 4 * 4
    off = np.zeros(n, np.int64)
    if n > 1:
        np.cumsum(region[:-1], out=off[1:])
    pool_len = int(off[-1] + region[-1]) if n else 0
    pu8 = np.zeros(_pad16(pool_len) + 16, np.uint8) if u8 else None
    p2 = np.zeros(_pad16((pool_len + 3) // 4) + 16, np.uint8) if two_bit else None
    if n > 0 and (u8 or two_bit):
        args = (off.ctypes.data_as(P(ctypes.c_int64)), pu8.ctypes.data_as(P(ctypes.c_uint8)) if u8 else None,
                p2.ctypes.data_as(P(ctypes.c_uint8)) if two_bit else None, n_threads)
        st = (lib.gen_bases(ctypes.byref(cfg), *args) if idx is None else
              lib.gen_bases_idx(ctypes.byref(cfg), ip, *args))
        if st != 0:
            raise RuntimeError("gen_bases failed")
    b = Batch(w, pair_base, off, ql, off + ql, tl, qs, ts, pool_len, pu8, p2)
    if idx is not None:
        b.meta["indices"] = idx
    return b


def lengths(w: Workload, n_pairs: int | None = None, pair_base: int = 0, n_threads: int | None = None):
    """(q_len, t_len, q_seed, t_seed) of pairs [pair_base, pair_base + n_pairs)
    without the pools (pass 1 only: what a partitioner needs)."""
    n = w.n_pairs if n_pairs is None else int(n_pairs)
    if n_threads is None:
        n_threads = len(os.sched_getaffinity(0))
    cfg = _Cfg(w.seed, n, pair_base, w.mode, w.tlen_min, w.tlen_max, w.err, w.k, w.spurious,
               w.len_lo, w.len_hi, w.burst)
    out = [np.zeros(n, np.int32) for _ in range(4)]
    if n > 0:
        P = ctypes.POINTER
        st = _load().gen_lengths(ctypes.byref(cfg), *[a.ctypes.data_as(P(ctypes.c_int32)) for a in out],
                                 n_threads)
        if st != 0:
            raise RuntimeError("gen_lengths failed")
    return tuple(out)


def decode_2bit(pool: np.ndarray, start: int, length: int) -> bytes:
    """ACGT text of ``length`` bases from a 2-bit pool (test helper)."""
    idx = np.arange(start, start + length, dtype=np.int64)
    codes = (pool[idx >> 2] >> (2 * (idx & 3)).astype(np.uint8)) & 3
    return bytes(np.frombuffer(b"ACGT", np.uint8)[codes])


def pack_2bit(text: bytes | str) -> np.ndarray:
    """Pack an ACGT string into the 2-bit pool format (test helper), padded."""
    if isinstance(text, str):
        text = text.encode()
    lut = np.full(256, 255, np.uint8)
    for c, v in zip(b"ACGT", range(4)):
        lut[c] = v
    codes = lut[np.frombuffer(text, np.uint8)]
    if (codes == 255).any():
        raise ValueError("2-bit pool holds A/C/G/T only")
    out = np.zeros(_pad16((len(codes) + 3) // 4) + 16, np.uint8)
    for s in range(4):
        part = codes[s::4].astype(np.uint8) << (2 * s)
        out[:len(part)] |= part
    return out


def from_strings(pairs, k: int, w: Workload | None = None) -> Batch:
    """Build a Batch from explicit (q, t, qs, ts) tuples (test helper)."""
    w = w or Workload("explicit", len(pairs), k=k)
    w = w.with_(k=k, n_pairs=len(pairs))
    qs_, ts_, ql_, tl_, qo_, to_ = [], [], [], [], [], []
    text = bytearray()
    for q, t, a, b in pairs:
        q = q.encode() if isinstance(q, str) else bytes(q)
        t = t.encode() if isinstance(t, str) else bytes(t)
        qo_.append(len(text)); text += q; to_.append(len(text)); text += t
        while len(text) % 4:
            text += b"A"
        ql_.append(len(q)); tl_.append(len(t)); qs_.append(a); ts_.append(b)
    pool_len = len(text)
    pu8 = np.zeros(_pad16(pool_len) + 16, np.uint8)
    pu8[:pool_len] = np.frombuffer(bytes(text), np.uint8)
    try:
        p2 = pack_2bit(bytes(text))
    except ValueError:
        p2 = None
    return Batch(w, 0, np.array(qo_, np.int64), np.array(ql_, np.int32), np.array(to_, np.int64),
                 np.array(tl_, np.int32), np.array(qs_, np.int32), np.array(ts_, np.int32),
                 pool_len, pu8, p2)


# ---------------------------------------------------------------------------
# Protein-like pairs for the substitution-matrix generalisation (SURVEY.md §8f
# row 4; the paper names protein alignment as future work). Pure numpy,
# counter-based per pair like the DNA generator: pair p depends only on
# (seed, p). Holds none of the method's arithmetic: the matrix below is an
# INPUT of the method (like match / mismatch), not a computation of it.
PROTEIN_ALPHABET = 20
PROTEIN_SEED = SEED_BASE + 7


def protein_matrix(seed: int = PROTEIN_SEED) -> np.ndarray:
    """A synthetic symmetric 20 x 20 substitution matrix shaped like the
    BLOSUM family (NOT BLOSUM itself): diagonal 4..11, off-diagonal -4..1."""
    rng = np.random.default_rng(seed)
    off = np.triu(rng.integers(-4, 2, size=(PROTEIN_ALPHABET, PROTEIN_ALPHABET)), 1)
    m = off + off.T
    m[np.diag_indices(PROTEIN_ALPHABET)] = rng.integers(4, 12, PROTEIN_ALPHABET)
    return m.astype(np.int8)


def _mutate_protein(rng, t: np.ndarray, u: int, k: int, sub: float, indel: float) -> tuple[np.ndarray, int]:
    """One read from template t: per residue a substitution (prob sub), a
    deletion (indel/2) or an insertion after it (indel/2); residues [u, u+k)
    (the seed) are copied verbatim. Returns (read, read position of t[u])."""
    L = len(t)
    r = rng.random(L)
    subm = r < sub
    delm = (r >= sub) & (r < sub + indel / 2)
    insm = (r >= sub + indel / 2) & (r < sub + indel)
    subm[u:u + k] = delm[u:u + k] = insm[u:u + k] = False
    codes = t.copy()
    codes[subm] = (t[subm] + rng.integers(1, PROTEIN_ALPHABET, int(subm.sum()))) % PROTEIN_ALPHABET
    vals = np.stack([codes, rng.integers(0, PROTEIN_ALPHABET, L)], 1)
    mask = np.stack([~delm, insm], 1)
    read = vals[mask].astype(np.uint8)
    return read, int(mask.ravel()[:2 * u].sum())


def protein_pairs(n_pairs: int, len_lo: int = 200, len_hi: int = 1000, sub: float = 0.15,
                  indel: float = 0.02, k: int = 6, seed: int = PROTEIN_SEED, pair_base: int = 0,
                  xdrop: int = 50, gap: int = -4) -> Batch:
    """Homologous protein-like pairs: template length uniform in [len_lo,
    len_hi], residues uniform over 20 codes; each read = mutate(template) with
    substitution rate ``sub`` and indel rate ``indel`` per residue (so ~2x
    between the reads); seed = a k-mer copied verbatim into both reads. The u8
    pool holds codes 0..19 (not letters)."""
    w = Workload(f"protein_{len_lo}-{len_hi}_x{xdrop}", n_pairs, tlen_min=len_lo, tlen_max=len_hi,
                 err=2 * (sub + indel), k=k, match=0, mismatch=0, gap=gap, xdrop=xdrop, seed=seed)
    qs_, ts_, ql_, tl_, qo_, to_ = [], [], [], [], [], []
    parts = []
    off = 0
    for p in range(n_pairs):
        rng = np.random.default_rng([seed, pair_base + p])
        L = int(rng.integers(len_lo, len_hi + 1))
        t = rng.integers(0, PROTEIN_ALPHABET, L).astype(np.int64)
        u = int(rng.integers(0, L - k + 1))
        q, qs = _mutate_protein(rng, t, u, k, sub, indel)
        r, rs = _mutate_protein(rng, t, u, k, sub, indel)
        for read, pos, offs, lens, seeds in ((q, qs, qo_, ql_, qs_), (r, rs, to_, tl_, ts_)):
            pad = (-len(read)) % 4
            offs.append(off); lens.append(len(read)); seeds.append(pos)
            parts.append(read); parts.append(np.zeros(pad, np.uint8))
            off += len(read) + pad
    pool_len = off
    pu8 = np.zeros(_pad16(pool_len) + 16, np.uint8)
    if parts:
        pu8[:pool_len] = np.concatenate(parts)
    return Batch(w, pair_base, np.array(qo_, np.int64), np.array(ql_, np.int32), np.array(to_, np.int64),
                 np.array(tl_, np.int32), np.array(qs_, np.int32), np.array(ts_, np.int32), pool_len, pu8, None,
                 meta={"alphabet": PROTEIN_ALPHABET})


# ---------------------------------------------------------------------------
# A read SET for the BELLA-like many-to-many shell (
# PAPER.md §V). Pure numpy, seeded: a random genome, reads cut at
# uniform positions with log-uniform lengths, each mutated at e/2 (1/3
# substitution, 1/3 insertion after the base, 1/3 deletion; as gen.c), forward
# strand only. Holds none of the method's arithmetic.
READSET_SEED = SEED_BASE + 8


@dataclass
class ReadSet:
    n_reads: int
    off: np.ndarray       # int64 pool offset of every read (multiple of 4)
    len: np.ndarray       # int32 read lengths
    g_start: np.ndarray   # genome interval each read was cut from (ground truth)
    g_end: np.ndarray
    pool_len: int
    pool_u8: np.ndarray
    pool_2bit: np.ndarray
    codes: np.ndarray     # 2-bit code of every pool position (A=0 C=1 G=2 T=3)
    err: float
    coverage: float


def _mutate_dna(rng, t: np.ndarray, rate: float) -> np.ndarray:
    L = len(t)
    r = rng.random(L)
    subm = r < rate / 3
    delm = (r >= rate / 3) & (r < 2 * rate / 3)
    insm = (r >= 2 * rate / 3) & (r < rate)
    codes = t.copy()
    codes[subm] = (t[subm] + rng.integers(1, 4, int(subm.sum()))) % 4
    vals = np.stack([codes, rng.integers(0, 4, L)], 1)
    mask = np.stack([~delm, insm], 1)
    return vals[mask].astype(np.uint8)


def read_set(n_reads: int = 400, genome_len: int = 200_000, len_lo: int = 2000, len_hi: int = 8000,
             err: float = 0.15, repeats: int = 0, repeat_len: int = 400, seed: int = READSET_SEED) -> ReadSet:
    """Reads sampled from one random genome (BELLA-like input, synthetic).
    ``repeats`` families of two identical copies of a ``repeat_len`` block are
    planted at random genome positions: reads covering different copies share
    k-mers without overlapping (the false candidates BELLA's threshold rejects)."""
    rng = np.random.default_rng(seed)
    genome = rng.integers(0, 4, genome_len).astype(np.uint8)
    for _ in range(repeats):
        unit = rng.integers(0, 4, repeat_len).astype(np.uint8)
        for p in rng.integers(0, genome_len - repeat_len, 2):
            genome[p:p + repeat_len] = unit
    lens = np.exp(rng.uniform(math.log(len_lo), math.log(len_hi), n_reads)).astype(np.int64)
    starts = rng.integers(0, np.maximum(genome_len - lens, 1))
    reads = [_mutate_dna(np.random.default_rng([seed, r]), genome[starts[r]:starts[r] + lens[r]], err / 2)
             for r in range(n_reads)]
    rl = np.array([len(x) for x in reads], np.int64)
    region = (rl + 3) // 4 * 4
    off = np.zeros(n_reads, np.int64)
    if n_reads > 1:
        np.cumsum(region[:-1], out=off[1:])
    pool_len = int(off[-1] + region[-1]) if n_reads else 0
    codes = np.zeros(_pad16(pool_len) + 16, np.uint8)
    for r in range(n_reads):
        codes[off[r]:off[r] + rl[r]] = reads[r]
    pu8 = np.frombuffer(b"ACGT", np.uint8)[codes]
    pu8[pool_len:] = 0
    p2 = np.zeros(_pad16((pool_len + 3) // 4) + 16, np.uint8)
    c = codes[:(pool_len + 3) // 4 * 4].reshape(-1, 4)
    p2[:len(c)] = c[:, 0] | (c[:, 1] << 2) | (c[:, 2] << 4) | (c[:, 3] << 6)
    return ReadSet(n_reads, off, rl.astype(np.int32), starts.astype(np.int64), (starts + lens).astype(np.int64),
                   pool_len, pu8, p2, codes, err, float(lens.sum()) / genome_len)
