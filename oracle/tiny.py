"""Pure-Python helpers for pinning the C oracle on tiny inputs.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

* :func:`full_dp` -- the textbook full-matrix semi-global prefix DP of eq. P:85
  (§III-A) with no pruning: S(0,0) = 0, S(i,0) = i*gap,
  S(0,j) = j*gap, interior cells the max of the three moves.  With X = inf the
  X-drop sweep must reproduce it exactly (best = max(0, max S), argmax by the
  smallest antidiagonal then the smallest i, cells = m*n).  This is an
  independent algorithm (row-major full matrix, no live flags, no band), so it
  pins the recurrence, the argmax convention and the cell count.
* :func:`xdrop_dict` -- the X-drop definition executed literally over a dict of
  live cells, antidiagonal by antidiagonal, visiting every cell of the
  antidiagonal (no band).  It is a second reading of the same definition, used
  as a cross-check of the C oracle's band restriction on many random tiny
  cases; it is NOT counted as a pin.
"""
from __future__ import annotations


def full_dp(A, B, match: int = 1, mismatch: int = -1, gap: int = -1, subst=None):
    """Full prefix DP matrix (m+1) x (n+1) as a list of lists (eq. P:85).
    With ``subst`` (a square matrix indexed by symbol codes) the substitution
    score is subst[a_i][b_j] instead of match / mismatch."""
    m, n = len(A), len(B)
    S = [[0] * (n + 1) for _ in range(m + 1)]
    for i in range(1, m + 1):
        S[i][0] = i * gap
    for j in range(1, n + 1):
        S[0][j] = j * gap
    for i in range(1, m + 1):
        for j in range(1, n + 1):
            if subst is not None:
                s = subst[A[i - 1]][B[j - 1]]
            else:
                s = match if A[i - 1] == B[j - 1] else mismatch
            S[i][j] = max(S[i - 1][j - 1] + s, S[i][j - 1] + gap, S[i - 1][j] + gap)
    return S


def full_dp_best(A, B, match: int = 1, mismatch: int = -1, gap: int = -1, subst=None):
    """(best, i*, j*) of the unpruned prefix alignment: best = max(0, max S);
    argmax = the cell with S = best on the smallest antidiagonal i+j, then the
    smallest i; (0, 0) when best = 0 (the empty alignment)."""
    S = full_dp(A, B, match, mismatch, gap, subst)
    m, n = len(A), len(B)
    best, bi, bj = 0, 0, 0
    for d in range(0, m + n + 1):
        for i in range(max(0, d - n), min(m, d) + 1):
            j = d - i
            if S[i][j] > best:
                best, bi, bj = S[i][j], i, j
    return best, bi, bj


def xdrop_dict(A: str, B: str, X: int, match: int = 1, mismatch: int = -1, gap: int = -1,
               compat: bool = False):
    """Literal X-drop over a dict of live cells -> (best, i*, j*, cells).
    ``compat``: the SeqAn-compat reading (oracle header step 6): strict ``>`` on
    boundary cells for d >= 2, and (i*, j*) = the best live cell (smallest i) of
    the last antidiagonal with a live cell."""
    m, n = len(A), len(B)
    if compat and (m == 0 or n == 0):
        return 0, 0, 0, 0  # empty extension (c-amb-13)
    live = {0: {0: 0}}  # d -> {i: S}
    best, bi, bj = 0, 0, 0
    last = (0, 0)  # compat: the origin unless a later antidiagonal has a live cell
    cells = 0
    d = 0
    while True:
        d += 1
        p1 = live.get(d - 1, {})
        p2 = live.get(d - 2, {})
        if d >= 2 and (p1 or p2):
            los, his = [], []
            if p1:
                los.append(min(p1))
                his.append(max(p1) + 1)
            if p2:
                los.append(min(p2) + 1)
                his.append(max(p2) + 1)
            lo = max(1, d - n, min(los))
            hi = min(m, d - 1, max(his))
            cells += max(0, hi - lo + 1)
        thr = best - X
        cur = {}
        for i in range(max(0, d - n), min(m, d) + 1):
            j = d - i
            cand = []
            if i >= 1 and j >= 1 and (i - 1) in p2:
                cand.append(p2[i - 1] + (match if A[i - 1] == B[j - 1] else mismatch))
            if j >= 1 and i in p1:
                cand.append(p1[i] + gap)
            if i >= 1 and (i - 1) in p1:
                cand.append(p1[i - 1] + gap)
            boundary = compat and d >= 2 and (i == 0 or j == 0)
            if cand and (max(cand) > thr if boundary else max(cand) >= thr):
                cur[i] = max(cand)
        live[d] = cur
        if cur:
            v = max(cur.values())
            if v > best:
                best = v
                bi = min(i for i, s in cur.items() if s == v)
                bj = d - bi
            li = min(i for i, s in cur.items() if s == v)
            last = (li, d - li)
        if not cur and not p1:
            break
    if compat:
        bi, bj = last if d > 0 and any(live.values()) else (0, 0)
    return best, bi, bj, cells
