/*
 * xdrop_oracle.c — the CPU ORACLE for LOGAN's X-drop seed-and-extend
 * (Zeni et al., arXiv 2002.05200).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2002_05200_b200/csrc/); neither side includes the other.
 *
 * Plain, slow, obviously correct: int64 arithmetic, one array per antidiagonal
 * indexed by the query offset i, an explicit live flag per cell, no sentinel
 * values, no rings, no packing, no SIMD. Citations are PAPER.md lines
 * ("P:<line>") and the readings "c-amb-N" listed in DESIGN.md §3.
 *
 * Extension E(A, B, X; match, mismatch, gap), A = a_1..a_m, B = b_1..b_n:
 *  (1) cell (0,0) is live with S = 0; best = 0                (Alg. 1 l.2)
 *  (2) for d = 1, 2, ... every cell (i, j), i + j = d, 0<=i<=m, 0<=j<=n:
 *        C = { S(i-1,j-1) + (a_i == b_j ? match : mismatch)  if i,j >= 1 and live(i-1,j-1),
 *              S(i,j-1) + gap                                if j >= 1 and live(i,j-1),
 *              S(i-1,j) + gap                                if i >= 1 and live(i-1,j) }
 *                                                             (eq. P:85 as a max, c-amb-1/2)
 *        C empty -> the cell is dead ("-inf, no longer considered")
 *        else S(i,j) = max C, live iff S(i,j) >= best_{d-1} - X  (Alg. 2 l.9, c-amb-4/5)
 *        best_d = max(best_{d-1}, max live S on d)
 *  (3) stop after the first d at which antidiagonals d and d-1 have no live
 *      cell (band empty, c-amb-7)
 *  (3b) optional Z-drop (minimap2's heuristic, which the paper names as an
 *      X-drop variant; reading c-amb-19): after antidiagonal d (best
 *      already updated), stop if best - M_d > Z + |gap| * |(i_d - i*) - (j_d - j*)|
 *      where M_d is the largest live score on d at (i_d, j_d), smallest i
 *  (4) result: best; (i*, j*) = the live cell with S = best on the smallest d,
 *      smallest i on that d; (0,0) if best = 0                 (c-amb-8, c-amb-9)
 *  (5) cells = sum over d >= 2 of |[lo_d, hi_d]| with
 *        lo_d = max(1, d-n, min(F_{d-1}, F_{d-2}+1)),
 *        hi_d = min(m, d-1, max(L_{d-1}, L_{d-2})+1),
 *      F_e / L_e = smallest / largest i over the live cells of antidiagonal e
 *      (boundary cells included; F_0 = L_0 = 0), only the terms of non-empty
 *      antidiagonals taken, empty band if both are empty     (c-amb-14)
 *
 *  (6) optional SeqAn-compat mode ([outside-PAPER] readings
 *      c-amb-24/25 of DESIGN.md §3, not verified against SeqAn, which is not
 *      available here): boundary cells (i = 0 or j = 0) on antidiagonals d >= 2
 *      are live only if S > best_{d-1} - X (strict; antidiagonal 1 keeps >=),
 *      and the returned cell is the "longest extension": the highest-scoring
 *      live cell (smallest i on ties) of the LAST antidiagonal that has a live
 *      cell, instead of the argmax of step (4); best is unchanged. An empty
 *      extension (m = 0 or n = 0) returns best 0 at (0,0) with 0 cells, as in
 *      the standard mode (c-amb-13; SeqAn returns at once for an empty segment).
 *
 * Step (2) visits, on antidiagonal d, only the columns that are adjacent to a
 * live cell of d-1 or d-2: a cell elsewhere has C = {} and is dead by
 * definition, so skipping it changes nothing. `full_scan = 1` visits every
 * column of the antidiagonal instead (tests check both give the same result).
 *
 * Substitution matrices (protein alignment is the paper's
 * future work): oracle_extend_subst / oracle_pairs_subst replace
 * "a_i == b_j ? match : mismatch" by subst[a_i * alph + b_j] and nothing else.
 *
 * Parity pins (tests/test_oracle_pins.py): brute-force full DP at X = inf,
 * closed forms (identical reads, disjoint alphabets, identical prefix + all
 * mismatch tail, X = 0 on identical reads), hand-worked examples
 * (tests/golden/), invariants (swap symmetry, 0 <= best <= full-DP value at
 * the argmax cell).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef struct {
    int64_t best;   /* final best ("return(best)")            */
    int64_t i, j;   /* argmax cell, extension-local                 */
    uint64_t cells; /* band cells (step 5)                          */
    int64_t last_d; /* antidiagonal at which the sweep stopped      */
} oracle_ext_t;

/* Result layout shared with nothing: the CUDA side has its own struct. */
typedef struct {
    int32_t score, q_begin, q_end, t_begin, t_end;
} oracle_pair_t;

#define ORACLE_OK 0
#define ORACLE_EINVAL 1
#define ORACLE_ENOMEM 2
#define ORACLE_ERANGE 3 /* a value did not fit int32 */

static int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
static int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

/*
 * One antidiagonal: value and live flag for each column i in [0, m].
 * lo/hi = smallest / largest live column, has_live = whether any is live.
 */
typedef struct {
    int64_t *val;
    uint8_t *live;
    int64_t lo, hi;  /* columns written on this antidiagonal (visited range) */
    int has_live;
    int64_t F, L;    /* smallest / largest live column                   */
} antidiag_t;

static int antidiag_init(antidiag_t *a, int64_t m) {
    a->val = (int64_t *)calloc((size_t)(m + 1), sizeof(int64_t));
    a->live = (uint8_t *)calloc((size_t)(m + 1), 1);
    a->lo = 0;
    a->hi = -1;
    a->has_live = 0;
    a->F = a->L = 0;
    return (a->val && a->live) ? 0 : -1;
}

static void antidiag_free(antidiag_t *a) {
    free(a->val);
    free(a->live);
}

/* live(i) on this antidiagonal: only columns that were visited can be live. */
static int is_live(const antidiag_t *a, int64_t i) {
    if (i < a->lo || i > a->hi) return 0;
    return a->live[i];
}

/* Clear the flags of the previously visited range before reuse. */
static void antidiag_clear(antidiag_t *a) {
    for (int64_t i = a->lo; i <= a->hi; ++i) a->live[i] = 0;
    a->lo = 0;
    a->hi = -1;
    a->has_live = 0;
}

/*
 * Substitution score s(a_i, b_j) of eq. P:85: match / mismatch, or, in the
 * substitution-matrix generalisation (protein alignment is
 * the paper's stated future work), the matrix entry subst[a * alph + b].
 */
static int64_t sub_score(uint8_t a, uint8_t b, int64_t match, int64_t mismatch,
                         const int8_t *subst, int64_t alph) {
    if (subst) return subst[(int64_t)a * alph + b];
    return a == b ? match : mismatch;
}

static int extend_impl(const uint8_t *A, int64_t m, const uint8_t *B, int64_t n,
                       int64_t match, int64_t mismatch, const int8_t *subst, int64_t alph,
                       int64_t gap, int64_t X, int64_t zdrop, int compat, int full_scan, oracle_ext_t *out);

int oracle_extend(const uint8_t *A, int64_t m, const uint8_t *B, int64_t n,
                  int64_t match, int64_t mismatch, int64_t gap, int64_t X,
                  int full_scan, oracle_ext_t *out) {
    return extend_impl(A, m, B, n, match, mismatch, NULL, 0, gap, X, -1, 0, full_scan, out);
}

/* The same extension with s(a, b) = subst[a * alph + b]; every code of A and B
 * must be < alph (ORACLE_EINVAL otherwise). */
int oracle_extend_subst(const uint8_t *A, int64_t m, const uint8_t *B, int64_t n,
                        const int8_t *subst, int64_t alph, int64_t gap, int64_t X,
                        int full_scan, oracle_ext_t *out) {
    if (!subst || alph < 1 || alph > 256) return ORACLE_EINVAL;
    for (int64_t i = 0; i < m; ++i) if (A[i] >= alph) return ORACLE_EINVAL;
    for (int64_t j = 0; j < n; ++j) if (B[j] >= alph) return ORACLE_EINVAL;
    return extend_impl(A, m, B, n, 0, 0, subst, alph, gap, X, -1, 0, full_scan, out);
}

/* The general extension: subst = NULL for match / mismatch, zdrop < 0 for no
 * Z-drop (otherwise step (3b) of the header applies). */
int oracle_extend_z(const uint8_t *A, int64_t m, const uint8_t *B, int64_t n,
                    int64_t match, int64_t mismatch, const int8_t *subst, int64_t alph,
                    int64_t gap, int64_t X, int64_t zdrop, int full_scan, oracle_ext_t *out) {
    if (subst) {
        if (alph < 1 || alph > 256) return ORACLE_EINVAL;
        for (int64_t i = 0; i < m; ++i) if (A[i] >= alph) return ORACLE_EINVAL;
        for (int64_t j = 0; j < n; ++j) if (B[j] >= alph) return ORACLE_EINVAL;
    }
    return extend_impl(A, m, B, n, match, mismatch, subst, alph, gap, X, zdrop, 0, full_scan, out);
}

/* SeqAn-compat mode (header step 6; match / mismatch scoring, optional Z-drop). */
int oracle_extend_compat(const uint8_t *A, int64_t m, const uint8_t *B, int64_t n,
                         int64_t match, int64_t mismatch, int64_t gap, int64_t X, int64_t zdrop,
                         int full_scan, oracle_ext_t *out) {
    return extend_impl(A, m, B, n, match, mismatch, NULL, 0, gap, X, zdrop, 1, full_scan, out);
}

static int extend_impl(const uint8_t *A, int64_t m, const uint8_t *B, int64_t n,
                       int64_t match, int64_t mismatch, const int8_t *subst, int64_t alph,
                       int64_t gap, int64_t X, int64_t zdrop, int compat, int full_scan, oracle_ext_t *out) {
    if (!out || m < 0 || n < 0 || X < 0 || (m > 0 && !A) || (n > 0 && !B)) return ORACLE_EINVAL;
    out->best = 0;
    out->i = 0;
    out->j = 0;
    out->cells = 0;
    out->last_d = 0;
    if (compat && (m == 0 || n == 0)) return ORACLE_OK; /* (6): empty extension */

    antidiag_t ad[3]; /* ad[d % 3] holds antidiagonal d */
    for (int k = 0; k < 3; ++k) {
        if (antidiag_init(&ad[k], m) != 0) {
            for (int q = 0; q <= k; ++q) antidiag_free(&ad[q]);
            return ORACLE_ENOMEM;
        }
    }

    /* (1) d = 0: the origin, live, S = 0; best = 0 (Alg. 1 l.2). */
    antidiag_t *a0 = &ad[0];
    a0->val[0] = 0;
    a0->live[0] = 1;
    a0->lo = a0->hi = 0;
    a0->has_live = 1;
    a0->F = a0->L = 0;
    int64_t best = 0, arg_i = 0, arg_j = 0;
    int64_t last_i = 0, last_j = 0; /* compat (step 6): the origin if nothing else is live */
    uint64_t cells = 0;
    /* antidiagonal -1 does not exist: treat it as empty */
    int prev2_exists = 0; /* whether antidiagonal d-2 exists (d >= 2) */

    int64_t d;
    for (d = 1;; ++d) {
        antidiag_t *cur = &ad[d % 3];
        antidiag_t *p1 = &ad[(d + 2) % 3]; /* d-1 */
        antidiag_t *p2 = &ad[(d + 1) % 3]; /* d-2 (stale if d < 2) */
        prev2_exists = (d >= 2);
        int p2_live = prev2_exists && p2->has_live;
        int p1_live = p1->has_live;

        /* cells on antidiagonal d: 0 <= i <= m, 0 <= j = d - i <= n */
        int64_t imin = max64(0, d - n), imax = min64(m, d);

        /* (5) band of interior cells for d >= 2 (c-amb-14). */
        if (d >= 2 && (p1_live || p2_live)) {
            int64_t lo, hi;
            if (p1_live && p2_live) {
                lo = min64(p1->F, p2->F + 1);
                hi = max64(p1->L, p2->L) + 1;
            } else if (p1_live) {
                lo = p1->F;
                hi = p1->L + 1;
            } else {
                lo = p2->F + 1;
                hi = p2->L + 1;
            }
            lo = max64(lo, max64(1, d - n));
            hi = min64(hi, min64(m, d - 1));
            if (hi >= lo) cells += (uint64_t)(hi - lo + 1);
        }

        /* (2) which columns to visit. */
        int64_t vlo, vhi;
        if (full_scan) {
            vlo = imin;
            vhi = imax;
        } else {
            /* a cell can have a live predecessor only at columns
             * [F_{d-1}, L_{d-1}+1] (up at i, left at i-1) or
             * [F_{d-2}+1, L_{d-2}+1] (diag at i-1)                        */
            vlo = INT64_MAX;
            vhi = INT64_MIN;
            if (p1_live) {
                vlo = min64(vlo, p1->F);
                vhi = max64(vhi, p1->L + 1);
            }
            if (p2_live) {
                vlo = min64(vlo, p2->F + 1);
                vhi = max64(vhi, p2->L + 1);
            }
            vlo = max64(vlo, imin);
            vhi = min64(vhi, imax);
        }

        /* threshold from the best at the END of antidiagonal d-1 (c-amb-5) */
        int64_t threshold = best - X;
        antidiag_clear(cur);
        int64_t dmax = 0;
        int have_max = 0;
        int64_t dmax_i = 0;
        if (vlo <= vhi) {
            cur->lo = vlo;
            cur->hi = vhi;
        }
        for (int64_t i = vlo; i <= vhi; ++i) {
            int64_t j = d - i;
            int have = 0;
            int64_t v = 0;
            /* diagonal predecessor (i-1, j-1) on d-2 */
            if (i >= 1 && j >= 1 && prev2_exists && is_live(p2, i - 1)) {
                int64_t s = sub_score(A[i - 1], B[j - 1], match, mismatch, subst, alph);
                int64_t c = p2->val[i - 1] + s;
                if (!have || c > v) v = c;
                have = 1;
            }
            /* up predecessor (i, j-1) on d-1 */
            if (j >= 1 && is_live(p1, i)) {
                int64_t c = p1->val[i] + gap;
                if (!have || c > v) v = c;
                have = 1;
            }
            /* left predecessor (i-1, j) on d-1 */
            if (i >= 1 && is_live(p1, i - 1)) {
                int64_t c = p1->val[i - 1] + gap;
                if (!have || c > v) v = c;
                have = 1;
            }
            int live = have && (v >= threshold); /* dropped iff S < best - X */
            /* (6) compat: boundary cells on d >= 2 need S > best - X */
            if (compat && d >= 2 && (i == 0 || j == 0)) live = have && (v > threshold);
            cur->live[i] = (uint8_t)live;
            cur->val[i] = live ? v : 0;
            if (live) {
                if (!cur->has_live) {
                    cur->F = i;
                    cur->has_live = 1;
                }
                cur->L = i;
                if (!have_max || v > dmax) { /* strict: first (smallest i) wins ties */
                    dmax = v;
                    dmax_i = i;
                    have_max = 1;
                }
            }
        }
        /* best updated only after the whole antidiagonal; argmax moves
         * only on a strict increase, so the earliest antidiagonal wins. */
        if (have_max && dmax > best) {
            best = dmax;
            arg_i = dmax_i;
            arg_j = d - dmax_i;
        }
        /* (6) compat: the best live cell of the last antidiagonal with a live cell */
        if (have_max) {
            last_i = dmax_i;
            last_j = d - dmax_i;
        }
        /* (3b) Z-drop (the variant the paper names; c-amb-19): stop after
         * antidiagonal d when best - M_d > Z + |gap| * |(i_d - i*) - (j_d - j*)|,
         * M_d / (i_d, j_d) = d's max live score and its cell (smallest i). */
        if (zdrop >= 0 && have_max) {
            int64_t off = (dmax_i - arg_i) - ((d - dmax_i) - arg_j);
            if (off < 0) off = -off;
            if (best - dmax > zdrop + (-gap) * off) break;
        }
        /* (3) termination: antidiagonals d and d-1 both empty */
        if (!cur->has_live && !p1->has_live) break;
        if (d > m + n + 2) break; /* cannot happen; defensive */
    }

    for (int k = 0; k < 3; ++k) antidiag_free(&ad[k]);
    out->best = best;
    out->i = compat ? last_i : arg_i;
    out->j = compat ? last_j : arg_j;
    out->cells = cells;
    out->last_d = d;
    return ORACLE_OK;
}

/* ---------------------------------------------------------------------- */
/* Pair level: seed split (Fig. 5) and result assembly.       */

/* base p of the pool as a byte: u8 = raw byte, 2-bit = code 0..3 */
static uint8_t pool_base(const uint8_t *pool, int fmt, int64_t p) {
    if (fmt == 0) return pool[p];
    return (uint8_t)((pool[p >> 2] >> (2 * (p & 3))) & 3);
}

/*
 * One pair. Left extension: A = reverse(q[0:qs)), B = reverse(t[0:ts)).
 * Right extension: A = q[qs+k:M), B = t[ts+k:N). seed_score = sum over the k
 * seed columns (c-amb-10). Coordinates per c-amb-8.
 */
static int pair_impl(const uint8_t *pool, int fmt, int64_t pool_len,
                     int64_t q_off, int64_t q_len, int64_t t_off, int64_t t_len,
                     int64_t qs, int64_t ts, int64_t k,
                     int64_t match, int64_t mismatch, const int8_t *subst, int64_t alph,
                     int64_t gap, int64_t X, int64_t zdrop, int compat, oracle_pair_t *res,
                     uint64_t *cells_out);

int oracle_pair(const uint8_t *pool, int fmt, int64_t pool_len,
                int64_t q_off, int64_t q_len, int64_t t_off, int64_t t_len,
                int64_t qs, int64_t ts, int64_t k,
                int64_t match, int64_t mismatch, int64_t gap, int64_t X,
                oracle_pair_t *res, uint64_t *cells_out) {
    return pair_impl(pool, fmt, pool_len, q_off, q_len, t_off, t_len, qs, ts, k, match, mismatch,
                     NULL, 0, gap, X, -1, 0, res, cells_out);
}

static int pair_impl(const uint8_t *pool, int fmt, int64_t pool_len,
                     int64_t q_off, int64_t q_len, int64_t t_off, int64_t t_len,
                     int64_t qs, int64_t ts, int64_t k,
                     int64_t match, int64_t mismatch, const int8_t *subst, int64_t alph,
                     int64_t gap, int64_t X, int64_t zdrop, int compat, oracle_pair_t *res,
                     uint64_t *cells_out) {
    res->score = INT32_MIN;
    res->q_begin = res->q_end = res->t_begin = res->t_end = -1;
    if (cells_out) *cells_out = 0;
    if (k < 0 || q_len < 0 || t_len < 0 || qs < 0 || ts < 0 || qs + k > q_len || ts + k > t_len ||
        q_off < 0 || t_off < 0 || q_off + q_len > pool_len || t_off + t_len > pool_len)
        return ORACLE_OK; /* invalid pair: invalid result, not an error */

    int64_t mL = qs, nL = ts, mR = q_len - qs - k, nR = t_len - ts - k;
    uint8_t *AL = (uint8_t *)malloc((size_t)(mL + 1));
    uint8_t *BL = (uint8_t *)malloc((size_t)(nL + 1));
    uint8_t *AR = (uint8_t *)malloc((size_t)(mR + 1));
    uint8_t *BR = (uint8_t *)malloc((size_t)(nR + 1));
    if (!AL || !BL || !AR || !BR) {
        free(AL); free(BL); free(AR); free(BR);
        return ORACLE_ENOMEM;
    }
    for (int64_t i = 1; i <= mL; ++i) AL[i - 1] = pool_base(pool, fmt, q_off + qs - i);
    for (int64_t j = 1; j <= nL; ++j) BL[j - 1] = pool_base(pool, fmt, t_off + ts - j);
    for (int64_t i = 1; i <= mR; ++i) AR[i - 1] = pool_base(pool, fmt, q_off + qs + k + i - 1);
    for (int64_t j = 1; j <= nR; ++j) BR[j - 1] = pool_base(pool, fmt, t_off + ts + k + j - 1);

    int64_t seed = 0;
    int bad_code = 0;
    for (int64_t u = 0; u < k; ++u) {
        const uint8_t a = pool_base(pool, fmt, q_off + qs + u), b = pool_base(pool, fmt, t_off + ts + u);
        if (subst && (a >= alph || b >= alph)) bad_code = 1;
        else seed += sub_score(a, b, match, mismatch, subst, alph);
    }

    oracle_ext_t L, R;
    int st = bad_code ? ORACLE_EINVAL : ORACLE_OK;
    if (st == ORACLE_OK) st = extend_impl(AL, mL, BL, nL, match, mismatch, subst, alph, gap, X, zdrop, compat, 0, &L);
    if (st == ORACLE_OK) st = extend_impl(AR, mR, BR, nR, match, mismatch, subst, alph, gap, X, zdrop, compat, 0, &R);
    free(AL); free(BL); free(AR); free(BR);
    if (st != ORACLE_OK) return st;

    int64_t score = seed + L.best + R.best;
    int64_t qb = qs - L.i, qe = qs + k + R.i, tb = ts - L.j, te = ts + k + R.j;
    if (score > INT32_MAX || score < INT32_MIN + 1) return ORACLE_ERANGE;
    res->score = (int32_t)score;
    res->q_begin = (int32_t)qb;
    res->q_end = (int32_t)qe;
    res->t_begin = (int32_t)tb;
    res->t_end = (int32_t)te;
    if (cells_out) *cells_out = L.cells + R.cells;
    return ORACLE_OK;
}

/* ---------------------------------------------------------------------- */
/* Batch driver: pair-level parallelism over host threads (each pair is    */
/* computed by the single-threaded routine above; dynamic chunks of 8).    */

typedef struct {
    const uint8_t *pool;
    int fmt;
    int64_t pool_len;
    const int64_t *q_off, *t_off;
    const int32_t *q_len, *t_len, *q_seed, *t_seed;
    int64_t n;
    int64_t k, match, mismatch, gap, X;
    const int8_t *subst;
    int64_t alph;
    int64_t zdrop;
    int compat;
    oracle_pair_t *out;
    uint64_t *cells;
    int64_t next; /* shared cursor */
    pthread_mutex_t mu;
    int status;
} batch_job_t;

static void *batch_worker(void *arg) {
    batch_job_t *job = (batch_job_t *)arg;
    for (;;) {
        pthread_mutex_lock(&job->mu);
        int64_t b = job->next;
        job->next += 8;
        pthread_mutex_unlock(&job->mu);
        if (b >= job->n) break;
        int64_t e = b + 8 < job->n ? b + 8 : job->n;
        for (int64_t p = b; p < e; ++p) {
            uint64_t c = 0;
            int st = pair_impl(job->pool, job->fmt, job->pool_len, job->q_off[p], job->q_len[p],
                               job->t_off[p], job->t_len[p], job->q_seed[p], job->t_seed[p],
                               job->k, job->match, job->mismatch, job->subst, job->alph, job->gap, job->X,
                               job->zdrop, job->compat, &job->out[p], &c);
            if (job->cells) job->cells[p] = c;
            if (st != ORACLE_OK) {
                pthread_mutex_lock(&job->mu);
                job->status = st;
                pthread_mutex_unlock(&job->mu);
            }
        }
    }
    return NULL;
}

static int pairs_impl(const uint8_t *pool, int fmt, int64_t pool_len,
                      const int64_t *q_off, const int32_t *q_len,
                      const int64_t *t_off, const int32_t *t_len,
                      const int32_t *q_seed, const int32_t *t_seed, int64_t n_pairs,
                      int64_t k, int64_t match, int64_t mismatch, const int8_t *subst, int64_t alph,
                      int64_t gap, int64_t X, int64_t zdrop, int compat, oracle_pair_t *out, uint64_t *cells,
                      int n_threads);

int oracle_pairs(const uint8_t *pool, int fmt, int64_t pool_len,
                 const int64_t *q_off, const int32_t *q_len,
                 const int64_t *t_off, const int32_t *t_len,
                 const int32_t *q_seed, const int32_t *t_seed, int64_t n_pairs,
                 int64_t k, int64_t match, int64_t mismatch, int64_t gap, int64_t X,
                 oracle_pair_t *out, uint64_t *cells, int n_threads) {
    return pairs_impl(pool, fmt, pool_len, q_off, q_len, t_off, t_len, q_seed, t_seed, n_pairs, k,
                      match, mismatch, NULL, 0, gap, X, -1, 0, out, cells, n_threads);
}

/* SeqAn-compat mode (header step 6): match / mismatch scoring, optional Z-drop. */
int oracle_pairs_compat(const uint8_t *pool, int fmt, int64_t pool_len,
                        const int64_t *q_off, const int32_t *q_len,
                        const int64_t *t_off, const int32_t *t_len,
                        const int32_t *q_seed, const int32_t *t_seed, int64_t n_pairs,
                        int64_t k, int64_t match, int64_t mismatch, int64_t gap, int64_t X, int64_t zdrop,
                        oracle_pair_t *out, uint64_t *cells, int n_threads) {
    return pairs_impl(pool, fmt, pool_len, q_off, q_len, t_off, t_len, q_seed, t_seed, n_pairs, k,
                      match, mismatch, NULL, 0, gap, X, zdrop, 1, out, cells, n_threads);
}

/* Pairs scored with a substitution matrix subst[alph * alph] (u8 pool of
 * codes < alph): seed score and both extensions use s(a, b) = subst[a*alph+b]. */
int oracle_pairs_subst(const uint8_t *pool, int64_t pool_len,
                       const int64_t *q_off, const int32_t *q_len,
                       const int64_t *t_off, const int32_t *t_len,
                       const int32_t *q_seed, const int32_t *t_seed, int64_t n_pairs,
                       int64_t k, const int8_t *subst, int64_t alph, int64_t gap, int64_t X,
                       oracle_pair_t *out, uint64_t *cells, int n_threads) {
    if (!subst || alph < 1 || alph > 256) return ORACLE_EINVAL;
    return pairs_impl(pool, 0, pool_len, q_off, q_len, t_off, t_len, q_seed, t_seed, n_pairs, k,
                      0, 0, subst, alph, gap, X, -1, 0, out, cells, n_threads);
}

/* The general batch: subst = NULL for match / mismatch (then fmt selects the
 * pool format), zdrop < 0 for no Z-drop. */
int oracle_pairs_z(const uint8_t *pool, int fmt, int64_t pool_len,
                   const int64_t *q_off, const int32_t *q_len,
                   const int64_t *t_off, const int32_t *t_len,
                   const int32_t *q_seed, const int32_t *t_seed, int64_t n_pairs,
                   int64_t k, int64_t match, int64_t mismatch, const int8_t *subst, int64_t alph,
                   int64_t gap, int64_t X, int64_t zdrop, oracle_pair_t *out, uint64_t *cells, int n_threads) {
    if (subst && (alph < 1 || alph > 256 || fmt != 0)) return ORACLE_EINVAL;
    return pairs_impl(pool, fmt, pool_len, q_off, q_len, t_off, t_len, q_seed, t_seed, n_pairs, k,
                      match, mismatch, subst, alph, gap, X, zdrop, 0, out, cells, n_threads);
}

static int pairs_impl(const uint8_t *pool, int fmt, int64_t pool_len,
                      const int64_t *q_off, const int32_t *q_len,
                      const int64_t *t_off, const int32_t *t_len,
                      const int32_t *q_seed, const int32_t *t_seed, int64_t n_pairs,
                      int64_t k, int64_t match, int64_t mismatch, const int8_t *subst, int64_t alph,
                      int64_t gap, int64_t X, int64_t zdrop, int compat, oracle_pair_t *out, uint64_t *cells,
                      int n_threads) {
    if (n_pairs < 0 || (n_pairs > 0 && (!pool || !q_off || !q_len || !t_off || !t_len || !q_seed ||
                                        !t_seed || !out)))
        return ORACLE_EINVAL;
    batch_job_t job = {pool, fmt, pool_len, q_off, t_off, q_len, t_len, q_seed, t_seed, n_pairs,
                       k, match, mismatch, gap, X, subst, alph, zdrop, compat, out, cells, 0,
                       PTHREAD_MUTEX_INITIALIZER, 0};
    if (n_threads < 1) n_threads = 1;
    if (n_threads == 1) {
        batch_worker(&job);
        return job.status;
    }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)n_threads);
    if (!th) return ORACLE_ENOMEM;
    for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, batch_worker, &job);
    for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
    free(th);
    return job.status;
}
