"""A BELLA-like many-to-many overlap shell around the X-drop batch.

PAPER.md §V integrates LOGAN into BELLA: k-mers are counted and
pruned, overlaps are detected by a sparse matrix product (read x k-mer times
its transpose), a seed k-mer is chosen per candidate pair by "binning" the
k-mer locations ("k-mer locations are used to estimate the overlap length and
to 'bin' k-mers to form a consensus"), the candidate pairs are aligned
as ONE batch on the GPU ("we modify BELLA to batch the entire set of
alignments together and send them to the GPU devices"), and an adaptive
threshold separates true overlaps from false positives.

The paper defines none of these stages beyond that sentence, so each is a
stated reading (readings 20-23), implemented plainly on the host
(numpy); only the alignment runs on the device, through ``api.xdrop_batch``
(or an injected ``aligner`` -- the tests inject the CPU oracle). Real data
sets (E. coli, C. elegans; Tables IV-V) stay out of scope: the reads come from
``datagen.read_set``.

* ``kmer_table``: every k-mer (2-bit code, forward strand) of every read with
  its position (reading 20: forward strand only; the synthetic reads have no
  reverse complements).
* reliable k-mers: occurrence count in [lo, hi] (reading 21: lo = 2 -- a
  k-mer seen once cannot seed an overlap; hi from the coverage -- k-mers seen
  far more often than the coverage predicts are repeats).
* ``candidate_pairs``: all read pairs sharing a reliable k-mer, with every
  shared k-mer's positions (the A * A^T SpGEMM, as a sort-and-group).
* ``choose_seeds``: the diagonal p_q - p_t of every shared k-mer is binned
  (width ``bin_width``); the most populated bin is the consensus, its median
  k-mer the seed (reading 22); the estimated overlap follows from the bin's
  diagonal and the read lengths.
* ``adaptive_keep``: keep a pair iff score >= rho * (1 - delta) * estimated
  overlap, rho the expected score per aligned base of a true overlap at the
  data's error rate (reading 23).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Overlaps:
    """The kept overlaps and everything the stages computed (host arrays)."""
    q: np.ndarray          # query read index of every candidate pair
    t: np.ndarray          # target read index
    q_seed: np.ndarray     # seed k-mer position in the query read
    t_seed: np.ndarray     # ... in the target read
    shared: np.ndarray     # shared reliable k-mers of the pair
    est_overlap: np.ndarray
    result: np.ndarray     # int32[n, 5]: score, q_begin, q_end, t_begin, t_end (the X-drop batch)
    cells: np.ndarray      # uint64[n]
    keep: np.ndarray       # bool[n]: passed the adaptive threshold
    stats: dict


def read_codes(reads, r: int) -> np.ndarray:
    """2-bit codes (A=0 C=1 G=2 T=3) of read r of a datagen.ReadSet."""
    return reads.codes[reads.off[r]:reads.off[r] + reads.len[r]]


def kmer_table(reads, k: int):
    """(kmer code uint64, read int32, position int32) of every k-mer of every read."""
    kms, rid, pos = [], [], []
    for r in range(reads.n_reads):
        c = read_codes(reads, r).astype(np.uint64)
        n = len(c) - k + 1
        if n <= 0:
            continue
        code = np.zeros(n, np.uint64)
        for u in range(k):  # code = sum_u c[i+u] * 4^(k-1-u)
            code = code * np.uint64(4) + c[u:u + n]
        kms.append(code)
        rid.append(np.full(n, r, np.int32))
        pos.append(np.arange(n, dtype=np.int32))
    if not kms:
        return np.zeros(0, np.uint64), np.zeros(0, np.int32), np.zeros(0, np.int32)
    return np.concatenate(kms), np.concatenate(rid), np.concatenate(pos)


def reliable_range(coverage: float, err: float, k: int) -> tuple[int, int]:
    """Reading 21: a true k-mer is seen about coverage * (1 - e/2)^k times (each
    read copy of it is error-free with that probability); the upper bound keeps
    counts up to three times that expectation plus 2 (repeats are pruned)."""
    expect = coverage * (1.0 - err / 2.0) ** k
    return 2, int(np.ceil(3.0 * expect)) + 2


def candidate_pairs(kmers, rid, pos, lo: int, hi: int):
    """Shared reliable k-mers of read pairs: arrays (q, t, pq, pt), q < t, one
    row per (pair, shared k-mer occurrence pair)."""
    order = np.lexsort((pos, rid, kmers))
    km, rd, ps = kmers[order], rid[order], pos[order]
    start = np.flatnonzero(np.r_[True, km[1:] != km[:-1]])
    cnt = np.diff(np.r_[start, len(km)])
    keep = (cnt >= lo) & (cnt <= hi)
    qs, ts, pqs, pts = [], [], [], []
    for g in np.unique(cnt[keep]):
        st = start[keep & (cnt == g)]
        idx = st[:, None] + np.arange(g)[None, :]       # rows: k-mer groups of size g
        R, Pp = rd[idx], ps[idx]
        for a in range(g):
            for b in range(a + 1, g):
                m = R[:, a] != R[:, b]
                ra, rb, pa, pb = R[m, a], R[m, b], Pp[m, a], Pp[m, b]
                sw = ra > rb
                qs.append(np.where(sw, rb, ra)); ts.append(np.where(sw, ra, rb))
                pqs.append(np.where(sw, pb, pa)); pts.append(np.where(sw, pa, pb))
    if not qs:
        z = np.zeros(0, np.int32)
        return z, z, z, z
    return (np.concatenate(qs).astype(np.int32), np.concatenate(ts).astype(np.int32),
            np.concatenate(pqs).astype(np.int32), np.concatenate(pts).astype(np.int32))


def choose_seeds(q, t, pq, pt, q_len, t_len, bin_width: int, min_shared: int = 1):
    """Reading 22 (BELLA's binning): per read pair, bin the diagonals
    pq - pt of its shared k-mers (width bin_width); the most populated bin is the
    consensus (ties: the lowest bin), its median k-mer (by query position) the
    seed. Returns per pair (q, t, q_seed, t_seed, shared k-mers, estimated
    overlap) for pairs with at least min_shared k-mers in the consensus bin."""
    if len(q) == 0:
        z = np.zeros(0, np.int32)
        return z, z, z, z, z, np.zeros(0, np.int64)
    diag = pq.astype(np.int64) - pt
    b = np.floor_divide(diag, bin_width)
    order = np.lexsort((pq, b, t, q))
    q, t, pq, pt, diag, b = q[order], t[order], pq[order], pt[order], diag[order], b[order]
    pair_key = q.astype(np.int64) * (1 << 31) + t
    bin_start = np.flatnonzero(np.r_[True, (pair_key[1:] != pair_key[:-1]) | (b[1:] != b[:-1])])
    bin_cnt = np.diff(np.r_[bin_start, len(q)])
    bin_pair = pair_key[bin_start]
    # the consensus bin of each pair: most k-mers, then the lowest bin (already sorted)
    o = np.lexsort((np.arange(len(bin_start)), -bin_cnt, bin_pair))
    first = np.r_[True, bin_pair[o][1:] != bin_pair[o][:-1]]
    best = o[first]
    s0, cnt = bin_start[best], bin_cnt[best]
    med = s0 + (cnt - 1) // 2
    sel = cnt >= min_shared
    med, cnt = med[sel], cnt[sel]
    qq, tt = q[med], t[med]
    d = diag[med]
    lq, lt = q_len[qq].astype(np.int64), t_len[tt].astype(np.int64)
    est = np.minimum(lq, d + lt) - np.maximum(0, d)  # the two reads' overlap on that diagonal
    return qq, tt, pq[med], pt[med], cnt.astype(np.int32), np.maximum(est, 0)


def adaptive_keep(score, est_overlap, rho: float, delta: float):
    """Reading 23: keep iff score >= rho (1 - delta) * estimated overlap."""
    return score >= np.floor(rho * (1.0 - delta) * est_overlap)


def run(reads, k: int = 17, xdrop: int = 50, match: int = 1, mismatch: int = -1, gap: int = -1,
        bin_width: int = 500, rho: float = 0.77, delta: float = 0.2, coverage: float | None = None,
        aligner=None, device=None) -> Overlaps:
    """The whole shell. ``aligner(batch, w) -> (int32[n,5], uint64[n])`` defaults
    to the CUDA path (``api.xdrop_batch`` on ``device``)."""
    import datagen
    cov = coverage if coverage is not None else reads.coverage
    lo, hi = reliable_range(cov, reads.err, k)
    kmers, rid, pos = kmer_table(reads, k)
    q, t, pq, pt = candidate_pairs(kmers, rid, pos, lo, hi)
    qq, tt, qs, ts, shared, est = choose_seeds(q, t, pq, pt, reads.len, reads.len, bin_width)
    w = datagen.Workload("bella_shell", len(qq), k=k, match=match, mismatch=mismatch, gap=gap, xdrop=xdrop)
    batch = datagen.Batch(w, 0, reads.off[qq].astype(np.int64), reads.len[qq].astype(np.int32),
                          reads.off[tt].astype(np.int64), reads.len[tt].astype(np.int32),
                          qs.astype(np.int32), ts.astype(np.int32), reads.pool_len, reads.pool_u8,
                          reads.pool_2bit)
    if aligner is None:
        res, cells = _gpu_align(batch, w, device)
    else:
        res, cells = aligner(batch, w)
    keep = adaptive_keep(res[:, 0], est, rho, delta) if len(qq) else np.zeros(0, bool)
    stats = {"reads": reads.n_reads, "kmers": int(len(kmers)), "reliable_range": [lo, hi],
             "candidate_pairs": int(len(qq)), "kept": int(keep.sum()),
             "cells": int(np.asarray(cells, np.uint64).sum())}
    return Overlaps(qq, tt, qs, ts, shared, est, res, np.asarray(cells, np.uint64), keep, stats)


def _gpu_align(batch, w, device):
    import torch

    from . import api
    if batch.n_pairs == 0:
        return np.zeros((0, 5), np.int32), np.zeros(0, np.uint64)
    db = api.to_device(batch, api._lib.LOGAN_SEQ_2BIT, device=device)
    out, cells = api.xdrop_batch(db, w.match, w.mismatch, w.gap, w.xdrop)
    torch.cuda.synchronize(db.q_len.device)
    return out.cpu().numpy(), cells.cpu().numpy().view(np.uint64)


def truth(reads, qq, tt, min_overlap: int):
    """Ground truth of the synthetic reads: the genome intervals of reads q and t
    overlap by at least min_overlap bases."""
    a0, a1 = reads.g_start[qq], reads.g_end[qq]
    b0, b1 = reads.g_start[tt], reads.g_end[tt]
    return (np.minimum(a1, b1) - np.maximum(a0, b0)) >= min_overlap


def all_true_pairs(reads, min_overlap: int) -> int:
    """Number of read pairs whose genome intervals overlap by >= min_overlap."""
    s, e = reads.g_start.astype(np.int64), reads.g_end.astype(np.int64)
    o = np.argsort(s)
    s, e = s[o], e[o]
    n = 0
    for i in range(len(s)):
        j = np.searchsorted(s, e[i] - min_overlap, side="right")  # later reads starting early enough
        if j > i + 1:
            ov = np.minimum(e[i], e[i + 1:j]) - s[i + 1:j]
            n += int((ov >= min_overlap).sum())
    return n
