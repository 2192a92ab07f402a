"""The BELLA-like shell (§V).

CPU: every host stage against a brute-force definition on small read sets,
and the whole shell with the CPU oracle as the aligner (separates true
overlaps from repeat-induced candidates). GPU: the shell with the CUDA path
gives exactly the oracle-aligned results (the aligner is the only difference).
"""
import itertools

import numpy as np
import pytest

import datagen
import oracle
from paper_2002_05200_b200 import bella


def _oracle_aligner(b, w):
    return oracle.pairs(b.pool_2bit, 1, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed, w.k, w.match,
                        w.mismatch, w.gap, w.xdrop, pool_len=b.pool_len)


def _small_set():
    return datagen.read_set(60, 30_000, 1500, 4000, repeats=8, repeat_len=300, seed=11)


def test_kmer_table_matches_naive():
    rs = datagen.read_set(6, 2000, 50, 200, seed=3)
    k = 7
    km, rid, pos = bella.kmer_table(rs, k)
    exp = []
    for r in range(rs.n_reads):
        c = bella.read_codes(rs, r)
        for p in range(len(c) - k + 1):
            exp.append((sum(int(c[p + u]) << (2 * (k - 1 - u)) for u in range(k)), r, p))
    assert sorted(zip(km.tolist(), rid.tolist(), pos.tolist())) == sorted(exp)


def test_candidate_pairs_match_brute_force():
    rs = datagen.read_set(12, 3000, 300, 900, seed=5)
    k = 9
    km, rid, pos = bella.kmer_table(rs, k)
    lo, hi = 2, 6
    q, t, pq, pt = bella.candidate_pairs(km, rid, pos, lo, hi)
    got = sorted(zip(q.tolist(), t.tolist(), pq.tolist(), pt.tolist()))
    occ = {}
    for a, r, p in zip(km.tolist(), rid.tolist(), pos.tolist()):
        occ.setdefault(a, []).append((r, p))
    exp = []
    for a, lst in occ.items():
        if lo <= len(lst) <= hi:
            for (r1, p1), (r2, p2) in itertools.combinations(lst, 2):
                if r1 != r2:
                    exp.append((r1, r2, p1, p2) if r1 < r2 else (r2, r1, p2, p1))
    assert got == sorted(exp)


def test_seed_choice_takes_the_consensus_bin():
    # pair (0, 1): three k-mers on diagonal ~100, one stray on diagonal 3000
    q = np.array([0, 0, 0, 0, 2], np.int32)
    t = np.array([1, 1, 1, 1, 3], np.int32)
    pq = np.array([150, 400, 3100, 700, 50], np.int32)
    pt = np.array([50, 300, 100, 610, 40], np.int32)
    lens = np.array([5000, 4000, 1000, 1000], np.int32)
    qq, tt, qs, ts, shared, est = bella.choose_seeds(q, t, pq, pt, lens, lens, 500)
    assert qq.tolist() == [0, 2] and tt.tolist() == [1, 3]
    assert (qs[0], ts[0], shared[0]) == (400, 300, 3)   # the median of the 3 consensus k-mers
    assert est[0] == min(5000, 100 + 4000) - 100         # diagonal 100: overlap [100, 4100) of read 0
    assert (qs[1], ts[1], shared[1], est[1]) == (50, 40, 1, 990)


def test_shell_with_oracle_separates_true_overlaps():
    rs = _small_set()
    ov = bella.run(rs, aligner=_oracle_aligner)
    tr = bella.truth(rs, ov.q, ov.t, 100)
    assert (~tr).sum() > 20  # the planted repeats give false candidates
    tp, fp = int((ov.keep & tr).sum()), int((ov.keep & ~tr).sum())
    assert tp / max(1, tr.sum()) > 0.95 and fp / max(1, ov.keep.sum()) < 0.1, (tp, fp, ov.stats)
    assert ov.stats["candidate_pairs"] == len(ov.q) and ov.stats["kept"] == int(ov.keep.sum())


@pytest.mark.gpu
def test_shell_gpu_equals_oracle():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2002_05200_b200 import build
    build.build()
    rs = _small_set()
    ref = bella.run(rs, aligner=_oracle_aligner)
    got = bella.run(rs)
    assert (got.q == ref.q).all() and (got.t == ref.t).all()
    assert (got.result == ref.result).all() and (got.cells == ref.cells).all() and (got.keep == ref.keep).all()
