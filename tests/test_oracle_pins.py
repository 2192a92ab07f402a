"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names the plausible oracle mistake it would catch.  Sources:
hand-worked fixtures (tests/golden/, derivations in DERIVATIONS.md), the
textbook full-matrix DP at X = inf (eq. P:85 with no pruning), closed forms
and provable invariants of the X-drop rule.
"""
import itertools
import os
import random

import numpy as np
import pytest

import datagen
import oracle
from oracle.tiny import full_dp, full_dp_best, xdrop_dict
from logan_testutil import read_tsv

INF = 10 ** 6


# ---------------------------------------------------------------- golden --
def test_golden_extensions(golden_dir):
    rows = read_tsv(os.path.join(golden_dir, "extensions.tsv"))
    assert len(rows) >= 7
    for (rid, A, B, X, ma, mi, g, best, i, j, cells, last_live) in rows:
        r = oracle.extend(A, B, int(X), int(ma), int(mi), int(g))
        assert (r.best, r.i, r.j, r.cells) == (int(best), int(i), int(j), int(cells)), rid
        assert r.last_d - 2 == int(last_live), rid
        rf = oracle.extend(A, B, int(X), int(ma), int(mi), int(g), full_scan=True)
        assert rf == r, rid


def test_golden_pairs(golden_dir):
    for (rid, q, t, qs, ts, k, X, ma, mi, g, score, qb, qe, tb, te, cells) in \
            read_tsv(os.path.join(golden_dir, "pairs.tsv")):
        res, c = oracle.pair(q, t, int(qs), int(ts), int(k), int(X), int(ma), int(mi), int(g))
        assert res == (int(score), int(qb), int(qe), int(tb), int(te)), rid
        assert c == int(cells), rid


# ------------------------------------------------ X = inf == full matrix DP --
def _all_strings(alphabet, maxlen):
    for L in range(0, maxlen + 1):
        for s in itertools.product(alphabet, repeat=L):
            yield "".join(s)


@pytest.mark.parametrize("scoring", [(1, -1, -1), (2, -3, -1), (1, -2, -3), (3, -1, -2)])
def test_xinf_equals_full_dp_exhaustive(scoring):
    """Catches: a dropped or mis-signed move, a wrong argmax convention, a
    wrong cell count (must be m*n when nothing is pruned)."""
    ma, mi, g = scoring
    strings = list(_all_strings("AC", 5))
    for A in strings:
        for B in strings:
            r = oracle.extend(A, B, INF, ma, mi, g)
            assert (r.best, r.i, r.j) == full_dp_best(A, B, ma, mi, g), (A, B)
            assert r.cells == len(A) * len(B), (A, B)


def test_xinf_equals_full_dp_random_dna():
    rng = random.Random(7)
    for _ in range(400):
        A = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 14)))
        B = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 14)))
        ma, mi, g = rng.randint(1, 5), -rng.randint(1, 5), -rng.randint(1, 5)
        r = oracle.extend(A, B, INF, ma, mi, g)
        assert (r.best, r.i, r.j) == full_dp_best(A, B, ma, mi, g)
        assert r.cells == len(A) * len(B)


# ------------------------------------------------------------ closed forms --
def test_identical_reads_closed_form():
    """Identical reads: score = M*match, coordinates [0, M) for any X >= 0 and
    any seed (the unique optimum is the full diagonal)."""
    rng = np.random.default_rng(11)
    for _ in range(60):
        M = int(rng.integers(17, 400))
        q = "".join(rng.choice(list("ACGT"), M))
        k = int(rng.integers(0, 18))
        qs = int(rng.integers(0, M - k + 1))
        X = int(rng.choice([0, 1, 3, 10, 50]))
        ma = int(rng.integers(1, 4))
        res, _ = oracle.pair(q, q, qs, qs, k, X, ma, -int(rng.integers(1, 4)), -int(rng.integers(1, 4)))
        assert res == (M * ma, 0, M, 0, M)


@pytest.mark.parametrize("scoring", [(2, -3, -1), (1, -2, -3), (3, -1, -2), (1, -1, -1)])
def test_identical_extension_x0_cells(scoring):
    """X = 0 on identical extensions: only the diagonal and its two side cells
    per antidiagonal are evaluated: cells = 3L - 2 (L >= 1)."""
    ma, mi, g = scoring
    for L in (1, 2, 3, 7, 40, 333):
        A = ("ACGTTGCA" * 60)[:L]
        r = oracle.extend(A, A, 0, ma, mi, g)
        assert (r.best, r.i, r.j) == (L * ma, L, L)
        assert r.cells == 3 * L - 2


@pytest.mark.parametrize("X", [0, 1, 2, 5, 9, 20])
def test_disjoint_alphabets(X):
    """A-only vs C-only, +1/-1/-1: S(i,j) = -max(i,j); live set {max(i,j) <= X};
    best 0 at (0,0); cells = (X+1)^2 when m, n > X; last live antidiagonal 2X.
    Catches: wrong boundary-cell rule, wrong band hull."""
    m = n = X + 7
    r = oracle.extend("A" * m, "C" * n, X)
    assert (r.best, r.i, r.j) == (0, 0, 0)
    assert r.cells == (X + 1) ** 2
    assert r.last_d - 2 == 2 * X


@pytest.mark.parametrize("p,X", [(1, 1), (5, 2), (12, 7), (30, 3), (8, 0)])
def test_identical_prefix_then_disjoint_tail(p, X):
    """Identical prefix of length p, then an all-mismatch tail: best p at (p,p)
    and the tail is explored to depth X (last live antidiagonal 2p + 2X)."""
    prefix = "".join(random.Random(p).choice("GT") for _ in range(p))  # tails share no base with it
    A = prefix + "A" * (X + 9)
    B = prefix + "C" * (X + 9)
    r = oracle.extend(A, B, X)
    assert (r.best, r.i, r.j) == (p, p, p)
    assert r.last_d - 2 == 2 * p + 2 * X


@pytest.mark.parametrize("X", [0, 1, 2, 3, 4, 7, 10])
def test_mismatch_diagonal_depth(X):
    """mismatch -2, gap -3 on A-only vs C-only: S(i,j) = -2 min(i,j) - 3|i-j|;
    the deepest live cell is (q,q) with q = floor(X/2), so the last live
    antidiagonal is 2*floor(X/2); antidiagonal 1 can be empty while 2 is not."""
    r = oracle.extend("A" * 30, "C" * 30, X, 1, -2, -3)
    assert (r.best, r.i, r.j) == (0, 0, 0)
    assert r.last_d - 2 == 2 * (X // 2)


def test_empty_extensions():
    for A, B in (("", ""), ("ACGT", ""), ("", "ACGT")):
        r = oracle.extend(A, B, 50)
        assert (r.best, r.i, r.j, r.cells) == (0, 0, 0, 0)


# --------------------------------------------------------------- invariants --
def test_invariants_random_tiny():
    """0 <= best <= S_full(i*, j*) <= max S_full; swap symmetry of best and
    cells; full scan == band-restricted scan; X >= (m+n)*max|w| == X = inf."""
    rng = random.Random(3)
    for _ in range(1500):
        A = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 12)))
        B = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 12)))
        X = rng.randint(0, 12)
        ma, mi, g = rng.randint(1, 3), -rng.randint(1, 3), -rng.randint(1, 3)
        r = oracle.extend(A, B, X, ma, mi, g)
        S = full_dp(A, B, ma, mi, g)
        assert 0 <= r.best <= S[r.i][r.j] <= max(0, max(max(row) for row in S))
        s = oracle.extend(B, A, X, ma, mi, g)
        assert (s.best, s.cells) == (r.best, r.cells)
        assert oracle.extend(A, B, X, ma, mi, g, full_scan=True) == r
        big = (len(A) + len(B)) * max(ma, -mi, -g)
        assert oracle.extend(A, B, big, ma, mi, g) == oracle.extend(A, B, INF, ma, mi, g)


def test_cross_check_python_dict_oracle():
    """Second reading of the definition (not a pin): dict-of-live-cells."""
    rng = random.Random(5)
    for _ in range(1500):
        A = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 10)))
        B = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 10)))
        X = rng.randint(0, 10)
        ma, mi, g = rng.randint(1, 3), -rng.randint(1, 3), -rng.randint(1, 3)
        r = oracle.extend(A, B, X, ma, mi, g)
        assert (r.best, r.i, r.j, r.cells) == xdrop_dict(A, B, X, ma, mi, g), (A, B, X)


def test_larger_x_can_lower_the_score():
    """BASELINE's "larger X never lowers the score" is false for X-drop
    (c-amb-16): a larger X lets an early branch raise best and kill the branch
    that would score higher.  Cross-checked against the dict oracle."""
    A, B = "AATCACCCTTGGCCCT", "ACTATCTGCCCCT"
    got = [oracle.extend(A, B, X) for X in (1, 2, 3)]
    assert [r.best for r in got] == [4, 3, 4]
    assert [xdrop_dict(A, B, X)[0] for X in (1, 2, 3)] == [4, 3, 4]
    # argmax and cells of SURVEY.md §8c c-amb-16's table (16 x 13: full DP 4 at (16,13), 208 cells)
    assert [(r.i, r.j, r.cells) for r in got] == [(16, 13, 64), (8, 11, 89), (16, 13, 123)]
    full = oracle.extend(A, B, INF)
    assert (full.best, full.i, full.j, full.cells) == (4, 16, 13, 208)
    assert full_dp_best(A, B, 1, -1, -1) == (4, 16, 13)


# ------------------------------------------------------------- pair level --
def test_pair_u8_equals_2bit_and_left_right_independent():
    w = datagen.CONFIGS[1]
    b = datagen.generate(w, n_pairs=64)
    args = (b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed, w.k, 1, -1, -1, 50)
    o8, c8 = oracle.pairs(b.pool_u8, 0, *args, pool_len=b.pool_len)
    o2, c2 = oracle.pairs(b.pool_2bit, 1, *args, pool_len=b.pool_len)
    assert (o8 == o2).all() and (c8 == c2).all()
    # pair assembly from two explicit extensions
    for p in range(8):
        q = datagen.decode_2bit(b.pool_2bit, b.q_off[p], b.q_len[p]).decode()
        t = datagen.decode_2bit(b.pool_2bit, b.t_off[p], b.t_len[p]).decode()
        qs, ts, k = int(b.q_seed[p]), int(b.t_seed[p]), w.k
        L = oracle.extend(q[:qs][::-1], t[:ts][::-1], 50)
        R = oracle.extend(q[qs + k:], t[ts + k:], 50)
        seed = sum(1 if q[qs + u] == t[ts + u] else -1 for u in range(k))
        assert tuple(o8[p]) == (seed + L.best + R.best, qs - L.i, qs + k + R.i, ts - L.j, ts + k + R.j)
        assert c8[p] == L.cells + R.cells
    # permutation of the batch permutes the results
    perm = np.random.default_rng(0).permutation(64)
    op, cp = oracle.pairs(b.pool_u8, 0, b.q_off[perm], b.q_len[perm], b.t_off[perm], b.t_len[perm],
                          b.q_seed[perm], b.t_seed[perm], w.k, 1, -1, -1, 50, pool_len=b.pool_len)
    assert (op == o8[perm]).all() and (cp == c8[perm]).all()


def test_invalid_pairs_get_invalid_result():
    b = datagen.from_strings([("ACGTACGT", "ACGTACGT", 2, 2)], k=3)
    bad = [  # (q_seed, t_seed, k)
        (-1, 2, 3), (2, -1, 3), (6, 2, 3), (2, 6, 3),
    ]
    for qs, ts, k in bad:
        o, c = oracle.pairs(b.pool_u8, 0, b.q_off, b.q_len, b.t_off, b.t_len, [qs], [ts], k,
                            1, -1, -1, 10, pool_len=b.pool_len)
        assert tuple(o[0]) == (-2 ** 31, -1, -1, -1, -1) and c[0] == 0
    # seed at the read ends: empty extensions on that side
    o, c = oracle.pairs(b.pool_u8, 0, b.q_off, b.q_len, b.t_off, b.t_len, [0], [0], 8,
                        1, -1, -1, 10, pool_len=b.pool_len)
    assert tuple(o[0]) == (8, 0, 8, 0, 8) and c[0] == 0


# ---------------------------------------------------------------------------
# Substitution-matrix generalisation

def test_subst_golden_s1():
    """Hand-worked example S1 (tests/golden/DERIVATIONS.md)."""
    M = [[3, -2, -1], [-2, 2, -3], [-1, -3, 1]]
    r = oracle.extend_subst(bytes([0, 1, 2]), bytes([0, 2, 1]), 2, M, -2)
    assert (r.best, r.i, r.j, r.cells) == (3, 1, 1, 9)


def test_subst_infinite_x_is_full_dp():
    """X = inf with a matrix equals the textbook full prefix DP with that matrix
    (exhaustive over all strings of length <= 3 on a 3-letter alphabet, a
    symmetric and an asymmetric matrix, two gap penalties)."""
    import itertools
    mats = [[[3, -2, -1], [-2, 2, -3], [-1, -3, 1]], [[2, -3, 1], [0, 4, -2], [-1, -1, 1]]]
    strs = [list(s) for L in range(4) for s in itertools.product(range(3), repeat=L)]
    for M in mats:
        for gap in (-1, -3):
            for A in strs:
                for B in strs:
                    r = oracle.extend_subst(bytes(A), bytes(B), 10 ** 6, M, gap)
                    best, bi, bj = full_dp_best(A, B, gap=gap, subst=M)
                    assert (r.best, r.i, r.j, r.cells) == (best, bi, bj, len(A) * len(B)), (A, B, M, gap)


def test_subst_reduces_to_match_mismatch():
    """The matrix M[a][b] = (a == b ? match : mismatch) gives exactly the pinned
    match / mismatch oracle, extension by extension and pair by pair."""
    rng = np.random.default_rng(7)
    for match, mismatch, gap in ((1, -1, -1), (2, -3, -1), (3, -1, -2)):
        M = [[match if a == b else mismatch for b in range(4)] for a in range(4)]
        for _ in range(60):
            A = rng.integers(0, 4, rng.integers(0, 40)).astype(np.uint8)
            B = A.copy() if rng.random() < 0.5 else rng.integers(0, 4, rng.integers(0, 40)).astype(np.uint8)
            if len(B) and rng.random() < 0.5:
                B[rng.integers(0, len(B), 3)] = rng.integers(0, 4, 3)
            X = int(rng.integers(0, 12))
            r1 = oracle.extend_subst(A.tobytes(), B.tobytes(), X, M, gap)
            r2 = oracle.extend(A.tobytes(), B.tobytes(), X, match, mismatch, gap)
            assert r1 == r2
    w = datagen.CONFIGS[1]
    b = datagen.generate(w, n_pairs=40)
    codes = np.frombuffer(bytes.maketrans(b"ACGT", bytes([0, 1, 2, 3])), np.uint8)[b.pool_u8]
    M = [[1 if a == c else -1 for c in range(4)] for a in range(4)]
    o1, c1 = oracle.pairs_subst(codes, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed, w.k, M, -1, 50,
                                pool_len=b.pool_len)
    o2, c2 = oracle.pairs(b.pool_u8, 0, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed, w.k,
                          1, -1, -1, 50, pool_len=b.pool_len)
    assert (o1 == o2).all() and (c1 == c2).all()


def test_subst_protein_invariants():
    """Protein-like pairs (datagen.protein_pairs): swap symmetry of best and
    cells for a symmetric matrix, 0 <= best <= full-DP value at the argmax, and
    codes outside the alphabet are rejected."""
    M = datagen.protein_matrix()
    b = datagen.protein_pairs(6, len_lo=30, len_hi=60)
    for p in range(b.n_pairs):
        q = b.pool_u8[b.q_off[p]:b.q_off[p] + b.q_len[p]]
        t = b.pool_u8[b.t_off[p]:b.t_off[p] + b.t_len[p]]
        for X in (5, 20, 60):
            r = oracle.extend_subst(q.tobytes(), t.tobytes(), X, M, -4)
            s = oracle.extend_subst(t.tobytes(), q.tobytes(), X, M, -4)
            assert (r.best, r.cells) == (s.best, s.cells)
            S = full_dp(list(q), list(t), gap=-4, subst=M.tolist())
            assert 0 <= r.best <= S[r.i][r.j]
    with pytest.raises(RuntimeError):
        oracle.extend_subst(bytes([0, 25]), bytes([1]), 5, M, -4)


# ---------------------------------------------------------------------------
# Z-drop (the X-drop variant the paper names; oracle header step 3b, c-amb-19)

def test_zdrop_closed_form():
    """Identical prefix of length p, then disjoint tails (A-only vs C/G-only), X
    unbounded: the antidiagonal maxima fall 1 per two antidiagonals on the
    diagonal, and the best off-diagonal cell trails by one |gap| on odd ones, so
    Z-drop stops after antidiagonal 2p + 2Z + 2 (for +1/-1/-1 and +1/-1/-2).
    Pins the '>' (not '>='), the antidiagonal max, and the |gap| * offset term:
    without the offset term (or with a multiplier of 1 at gap -2) the stop
    comes one antidiagonal earlier."""
    for gap in (-1, -2):
        for p in (0, 3, 10, 25):
            for Z in (0, 1, 2, 5, 9):
                A, B = "A" * p + "C" * 40, "A" * p + "G" * 40
                r = oracle.extend_z(A, B, 10 ** 6, Z, gap=gap)
                assert (r.best, r.i, r.j, r.last_d) == (p, p, p, 2 * p + 2 * Z + 2), (gap, p, Z, r)


def test_zdrop_off_or_unbounded_is_xdrop():
    """Z < 0 (off) and Z above any reachable drop reproduce the pinned X-drop
    oracle exactly, with and without a substitution matrix."""
    rng = np.random.default_rng(11)
    M = datagen.protein_matrix()
    for _ in range(80):
        A = rng.integers(0, 4, rng.integers(0, 60)).astype(np.uint8)
        B = A.copy() if rng.random() < 0.6 else rng.integers(0, 4, rng.integers(0, 60)).astype(np.uint8)
        if len(B):
            B[rng.integers(0, len(B), 4)] = rng.integers(0, 4, 4)
        X = int(rng.integers(0, 30))
        ref = oracle.extend(A.tobytes(), B.tobytes(), X)
        assert oracle.extend_z(A.tobytes(), B.tobytes(), X, -1) == ref
        assert oracle.extend_z(A.tobytes(), B.tobytes(), X, 10 ** 6) == ref
        refm = oracle.extend_subst(A.tobytes(), B.tobytes(), X, M, -4)
        assert oracle.extend_z(A.tobytes(), B.tobytes(), X, 10 ** 6, gap=-4, subst=M) == refm


def test_zdrop_truncates_the_xdrop_sweep():
    """With Z-drop the sweep is a prefix of the X-drop sweep: it stops no later,
    best and cells never exceed the X-drop values, and when it stops before the
    band empties the last antidiagonal satisfies the Z condition."""
    rng = np.random.default_rng(12)
    for _ in range(200):
        A = rng.integers(0, 4, rng.integers(1, 80)).astype(np.uint8)
        B = A.copy()
        B[rng.integers(0, len(B), max(1, len(B) // 5))] = rng.integers(0, 4, max(1, len(B) // 5))
        X, Z = int(rng.integers(5, 40)), int(rng.integers(0, 8))
        full = oracle.extend(A.tobytes(), B.tobytes(), X)
        z = oracle.extend_z(A.tobytes(), B.tobytes(), X, Z)
        assert z.last_d <= full.last_d and z.best <= full.best and z.cells <= full.cells
        if z.last_d == full.last_d:
            assert z == full


# ---------------------------------------------------------------------------
# SeqAn-compat mode (oracle header step 6; [outside-PAPER] readings c-amb-24/25)

def test_compat_golden(golden_dir):
    """Hand-worked compat extensions (tests/golden/compat.tsv, DERIVATIONS.md):
    C2 pins the strict boundary rule (the standard rule keeps (0,2) and reaches
    (1,3)), all three the longest-extension end cell."""
    rows = read_tsv(os.path.join(golden_dir, "compat.tsv"))
    assert len(rows) >= 3
    for (rid, A, B, X, ma, mi, g, best, i, j, cells, last_d) in rows:
        r = oracle.extend_compat(A, B, int(X), int(ma), int(mi), int(g))
        assert (r.best, r.i, r.j, r.cells, r.last_d) == (int(best), int(i), int(j), int(cells), int(last_d)), rid
        assert oracle.extend_compat(A, B, int(X), int(ma), int(mi), int(g), full_scan=True) == r, rid
    s = oracle.extend("A", "CCAA", 2)
    assert (s.best, s.i, s.j, s.cells) == (0, 0, 0, 4)  # the standard rule on C2


@pytest.mark.parametrize("scoring", [(1, -1, -1), (2, -3, -1)])
def test_compat_infinite_x_ends_at_the_corner(scoring):
    """X = inf: nothing drops, so the strict boundary rule changes nothing; best
    and cells are the full DP's, and the longest extension is the corner (m, n),
    the only cell of the last antidiagonal (an empty extension stays at (0,0))."""
    ma, mi, g = scoring
    for A in _all_strings("AC", 4):
        for B in _all_strings("AC", 4):
            r = oracle.extend_compat(A, B, INF, ma, mi, g)
            assert (r.best, r.cells) == (full_dp_best(A, B, ma, mi, g)[0], len(A) * len(B))
            assert (r.i, r.j) == ((len(A), len(B)) if A and B else (0, 0))  # empty extension: c-amb-13


@pytest.mark.parametrize("X", [1, 2, 3, 6, 9])
def test_compat_disjoint_alphabets(X):
    """A-only vs C-only (S = -max(i,j)): best 0, the last live antidiagonal is 2X
    holding only (X, X), cells (X+1)^2, as the standard rule."""
    m = X + 7
    r = oracle.extend_compat("A" * m, "C" * m, X)
    assert (r.best, r.i, r.j, r.cells, r.last_d) == (0, X, X, (X + 1) ** 2, 2 * X + 2)


def test_compat_cross_check_dict_reading():
    """Second reading (not a pin): the dict-of-live-cells model with the compat rules."""
    rng = random.Random(17)
    for _ in range(1500):
        A = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 10)))
        B = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 10)))
        X = rng.randint(0, 8)
        ma, mi, g = rng.randint(1, 3), -rng.randint(1, 3), -rng.randint(1, 3)
        r = oracle.extend_compat(A, B, X, ma, mi, g)
        assert (r.best, r.i, r.j, r.cells) == xdrop_dict(A, B, X, ma, mi, g, compat=True), (A, B, X)


def test_compat_pairs_assemble_extensions():
    w = datagen.CONFIGS[1]
    b = datagen.generate(w, n_pairs=24)
    o, c = oracle.pairs_compat(b.pool_u8, 0, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed, w.k,
                               1, -1, -1, 50, pool_len=b.pool_len)
    for p in range(6):
        q = datagen.decode_2bit(b.pool_2bit, b.q_off[p], b.q_len[p]).decode()
        t = datagen.decode_2bit(b.pool_2bit, b.t_off[p], b.t_len[p]).decode()
        qs, ts, k = int(b.q_seed[p]), int(b.t_seed[p]), w.k
        L = oracle.extend_compat(q[:qs][::-1], t[:ts][::-1], 50)
        R = oracle.extend_compat(q[qs + k:], t[ts + k:], 50)
        assert tuple(o[p]) == (k + L.best + R.best, qs - L.i, qs + k + R.i, ts - L.j, ts + k + R.j)
        assert c[p] == L.cells + R.cells
