/*
 * gen.c — seeded synthetic read-pair generator for the LOGAN X-drop workloads.
 *
 * Shared by the oracle tests and the CUDA path (it holds NONE of the method's
 * arithmetic: no scoring, no DP). Counter-based: pair p of a workload is a
 * pure function of (seed, p), so any pair or shard regenerates independently
 * of batching and of the number of GPUs.
 *
 * Workload recipe (the paper gives only "100K pairs, 2.5-7.5 kb,
 * about 15% error between the two reads", §VI-A):
 *  - mode 0 (template pairs, configs 1, 2, 3, 5): template T of length
 *    uniform in [tlen_min, tlen_max], i.i.d. uniform over ACGT; each read is
 *    mutate(T, e/2) independently (so the pairwise error is about e): per
 *    template base with probability e/2 an error event, one third each a
 *    substitution (uniform over the 3 other bases), an insertion of a random
 *    base after it, or a deletion. Seed: uniform over the template positions
 *    whose k bases are copied error-free and contiguously into both reads.
 *  - mode 1 (BELLA-like, config 4): a fraction `spurious` of pairs are two
 *    independent random reads (lengths log-uniform on [len_lo, len_hi]) with
 *    one identical random k-mer planted at a uniform position of each; the
 *    rest are dovetail overlaps: read lengths lq, lt log-uniform on
 *    [len_lo, len_hi], overlap o uniform on [len_lo, min(lq, lt)], reads cut
 *    from one template and mutated at e/2, seed a clean k-mer inside the
 *    overlap. Which read is the query is a fair coin.
 *  - burst (parity tests only): with probability `burst` per read, a random
 *    block of 50-300 bases is inserted at a uniform template position.
 *
 * Output is two passes over the pairs (lengths + seeds, then bases), both
 * parallel over pairs with pthreads. Bases are ASCII 'A','C','G','T' in the
 * u8 pool and codes 0..3 packed four per byte, LSB first, in the 2-bit pool.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    uint64_t seed;
    int64_t n_pairs;
    int64_t pair_base; /* global index of the first pair */
    int32_t mode;      /* 0 template pairs, 1 BELLA-like */
    int32_t tlen_min, tlen_max;
    double err;        /* pairwise error e */
    int32_t k;
    double spurious;
    int32_t len_lo, len_hi;
    double burst;
} gen_cfg_t;

/* ---- counter-based RNG: splitmix64 over a per-pair counter -------------- */
typedef struct {
    uint64_t s;
} rng_t;

static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static rng_t rng_for(uint64_t seed, uint64_t pair, uint64_t attempt) {
    rng_t r;
    r.s = mix64(seed ^ mix64(pair * 0x9e3779b97f4a7c15ULL + 0x632be59bd9b4e019ULL) ^
                mix64(attempt + 0x1234567ULL));
    return r;
}
static uint64_t next64(rng_t *r) {
    r->s += 0x9e3779b97f4a7c15ULL;
    return mix64(r->s);
}
static double unif(rng_t *r) { return (double)(next64(r) >> 11) * (1.0 / 9007199254740992.0); }
static uint32_t below(rng_t *r, uint32_t n) { return (uint32_t)(((next64(r) >> 32) * (uint64_t)n) >> 32); }
static int32_t log_uniform(rng_t *r, int32_t lo, int32_t hi) {
    double x = exp(log((double)lo) + unif(r) * (log((double)hi) - log((double)lo)));
    int32_t v = (int32_t)x;
    return v < lo ? lo : (v > hi ? hi : v);
}

/* ---- mutation with a template->read map (-1 = not copied verbatim) ------ */
static int64_t mutate(const uint8_t *T, int64_t L, double rate, double burst, rng_t *r,
                      uint8_t *out, int64_t *map) {
    int64_t len = 0;
    int64_t bpos = -1, blen = 0;
    if (burst > 0.0 && unif(r) < burst) {
        bpos = (int64_t)below(r, (uint32_t)L);
        blen = 50 + (int64_t)below(r, 251);
    }
    for (int64_t p = 0; p < L; ++p) {
        if (p == bpos)
            for (int64_t q = 0; q < blen; ++q) out[len++] = (uint8_t)below(r, 4);
        if (unif(r) < rate) {
            uint32_t type = below(r, 3);
            if (type == 0) { /* substitution */
                out[len++] = (uint8_t)((T[p] + 1 + below(r, 3)) & 3);
                map[p] = -1;
            } else if (type == 1) { /* insertion after the base */
                map[p] = len;
                out[len++] = T[p];
                out[len++] = (uint8_t)below(r, 4);
            } else { /* deletion */
                map[p] = -1;
            }
        } else {
            map[p] = len;
            out[len++] = T[p];
        }
    }
    return len;
}

/* clean seed start positions p in [lo, hi]: k template bases copied verbatim
 * and contiguously into both reads. Returns the chosen p or -1. */
static int64_t pick_seed(const int64_t *mq, const int64_t *mt, int64_t lo, int64_t hi, int32_t k,
                         rng_t *r) {
    int64_t count = 0;
    for (int pass = 0; pass < 2; ++pass) {
        int64_t target = pass ? (int64_t)below(r, (uint32_t)count) : -1;
        int64_t seen = 0;
        for (int64_t p = lo; p <= hi; ++p) {
            int ok = 1;
            for (int32_t u = 0; u < k && ok; ++u) {
                if (mq[p + u] < 0 || mt[p + u] < 0) ok = 0;
                else if (u > 0 && (mq[p + u] != mq[p] + u || mt[p + u] != mt[p] + u)) ok = 0;
            }
            if (ok) {
                if (pass && seen == target) return p;
                ++seen;
            }
        }
        if (!pass) {
            count = seen;
            if (count == 0) return -1;
        }
    }
    return -1;
}

/* Generate pair `gp` (global index) into q/t (capacity cap each). Returns 0. */
typedef struct {
    uint8_t *T, *q, *t;
    int64_t *mq, *mt;
    int64_t cap;
} scratch_t;

static int scratch_init(scratch_t *s, int64_t cap) {
    s->cap = cap;
    s->T = (uint8_t *)malloc((size_t)cap);
    s->q = (uint8_t *)malloc((size_t)cap * 2 + 512);
    s->t = (uint8_t *)malloc((size_t)cap * 2 + 512);
    s->mq = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
    s->mt = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
    return (s->T && s->q && s->t && s->mq && s->mt) ? 0 : -1;
}
static void scratch_free(scratch_t *s) {
    free(s->T); free(s->q); free(s->t); free(s->mq); free(s->mt);
}

static int64_t template_cap(const gen_cfg_t *c) {
    if (c->mode == 1) return 2 * (int64_t)c->len_hi + 16;
    return (int64_t)c->tlen_max + 16;
}

static void gen_pair(const gen_cfg_t *c, int64_t gp, scratch_t *s, int32_t *qlen, int32_t *tlen,
                     int32_t *qs, int32_t *ts) {
    double rate = c->err / 2.0;
    for (uint64_t attempt = 0;; ++attempt) {
        rng_t r = rng_for(c->seed, (uint64_t)gp, attempt);
        if (c->mode == 1 && unif(&r) < c->spurious) {
            int32_t lq = log_uniform(&r, c->len_lo, c->len_hi);
            int32_t lt = log_uniform(&r, c->len_lo, c->len_hi);
            for (int32_t i = 0; i < lq; ++i) s->q[i] = (uint8_t)below(&r, 4);
            for (int32_t i = 0; i < lt; ++i) s->t[i] = (uint8_t)below(&r, 4);
            int32_t a = (int32_t)below(&r, (uint32_t)(lq - c->k + 1));
            int32_t b = (int32_t)below(&r, (uint32_t)(lt - c->k + 1));
            for (int32_t u = 0; u < c->k; ++u) s->t[b + u] = s->q[a + u] = (uint8_t)below(&r, 4);
            *qlen = lq; *tlen = lt; *qs = a; *ts = b;
            return;
        }
        int64_t L, qa, qlen_t, ta, tlen_t, olo, ohi;
        if (c->mode == 1) {
            int32_t lq = log_uniform(&r, c->len_lo, c->len_hi);
            int32_t lt = log_uniform(&r, c->len_lo, c->len_hi);
            int32_t mn = lq < lt ? lq : lt;
            int32_t o = c->len_lo + (int32_t)below(&r, (uint32_t)(mn - c->len_lo + 1));
            L = (int64_t)lq + lt - o;
            qa = 0; qlen_t = lq; ta = lq - o; tlen_t = lt;
            olo = ta; ohi = lq - c->k;
        } else {
            L = c->tlen_min + (int64_t)below(&r, (uint32_t)(c->tlen_max - c->tlen_min + 1));
            qa = 0; qlen_t = L; ta = 0; tlen_t = L;
            olo = 0; ohi = L - c->k;
        }
        for (int64_t i = 0; i < L; ++i) s->T[i] = (uint8_t)below(&r, 4);
        int64_t lq = mutate(s->T + qa, qlen_t, rate, c->burst, &r, s->q, s->mq);
        int64_t lt = mutate(s->T + ta, tlen_t, rate, c->burst, &r, s->t, s->mt);
        /* seed in template coordinates p in [olo, ohi]; maps are per read */
        int64_t *mq = s->mq, *mt = s->mt;
        /* express both maps over template coordinates [olo, ohi+k) */
        int64_t cnt = ohi - olo + c->k;
        if (ohi < olo) continue;
        int64_t *tmpq = (int64_t *)malloc(sizeof(int64_t) * (size_t)cnt);
        int64_t *tmpt = (int64_t *)malloc(sizeof(int64_t) * (size_t)cnt);
        for (int64_t p = 0; p < cnt; ++p) {
            tmpq[p] = mq[olo + p - qa];
            tmpt[p] = mt[olo + p - ta];
        }
        int64_t p = pick_seed(tmpq, tmpt, 0, ohi - olo, c->k, &r);
        int64_t sq = p >= 0 ? tmpq[p] : -1, st = p >= 0 ? tmpt[p] : -1;
        free(tmpq);
        free(tmpt);
        if (p < 0) continue;
        int swap = (c->mode == 1) && (below(&r, 2) == 1);
        if (!swap) {
            *qlen = (int32_t)lq; *tlen = (int32_t)lt; *qs = (int32_t)sq; *ts = (int32_t)st;
        } else {
            /* exchange the roles: copy t into q's buffer via a rotation */
            uint8_t *tmp = s->q; s->q = s->t; s->t = tmp;
            *qlen = (int32_t)lt; *tlen = (int32_t)lq; *qs = (int32_t)st; *ts = (int32_t)sq;
        }
        return;
    }
}

/* ---- batch driver -------------------------------------------------------- */
typedef struct {
    const gen_cfg_t *cfg;
    int32_t *qlen, *tlen, *qs, *ts;
    const int64_t *off; /* pass 2: pair region start (bases) */
    uint8_t *u8;        /* may be NULL */
    uint8_t *b2;        /* may be NULL */
    const int64_t *idx; /* NULL: local pair p is global pair_base + p; else global idx[p] */
    int64_t next;
    pthread_mutex_t mu;
    int pass;
    int fail;
} job_t;

static const uint8_t ACGT[4] = {'A', 'C', 'G', 'T'};

static void *worker(void *arg) {
    job_t *j = (job_t *)arg;
    scratch_t s;
    int64_t cap = template_cap(j->cfg);
    if (scratch_init(&s, cap) != 0) {
        pthread_mutex_lock(&j->mu);
        j->fail = 1;
        pthread_mutex_unlock(&j->mu);
        return NULL;
    }
    for (;;) {
        pthread_mutex_lock(&j->mu);
        int64_t b = j->next;
        j->next += 16;
        pthread_mutex_unlock(&j->mu);
        if (b >= j->cfg->n_pairs) break;
        int64_t e = b + 16 < j->cfg->n_pairs ? b + 16 : j->cfg->n_pairs;
        for (int64_t p = b; p < e; ++p) {
            int32_t ql, tl, qs, ts;
            gen_pair(j->cfg, j->idx ? j->idx[p] : j->cfg->pair_base + p, &s, &ql, &tl, &qs, &ts);
            if (j->pass == 1) {
                j->qlen[p] = ql; j->tlen[p] = tl; j->qs[p] = qs; j->ts[p] = ts;
            } else {
                int64_t o = j->off[p];
                for (int32_t i = 0; i < ql + tl; ++i) {
                    uint8_t c = i < ql ? s.q[i] : s.t[i - ql];
                    int64_t pos = o + i;
                    if (j->u8) j->u8[pos] = ACGT[c];
                    if (j->b2) j->b2[pos >> 2] |= (uint8_t)(c << (2 * (pos & 3)));
                }
            }
        }
    }
    scratch_free(&s);
    return NULL;
}

static int run(job_t *j, int n_threads) {
    if (n_threads < 1) n_threads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)n_threads);
    if (!th) return -1;
    for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, worker, j);
    for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
    free(th);
    return j->fail ? -1 : 0;
}

/* Pass 1: lengths and seeds. */
int gen_lengths(const gen_cfg_t *cfg, int32_t *qlen, int32_t *tlen, int32_t *qs, int32_t *ts,
                int n_threads) {
    job_t j = {cfg, qlen, tlen, qs, ts, NULL, NULL, NULL, NULL, 0, PTHREAD_MUTEX_INITIALIZER, 1, 0};
    return run(&j, n_threads);
}

/* Pass 1 for an arbitrary set of global pair indices idx[0 .. cfg->n_pairs)
 * (a shard of a partitioned batch; pair_base is ignored). */
int gen_lengths_idx(const gen_cfg_t *cfg, const int64_t *idx, int32_t *qlen, int32_t *tlen, int32_t *qs,
                    int32_t *ts, int n_threads) {
    job_t j = {cfg, qlen, tlen, qs, ts, NULL, NULL, NULL, idx, 0, PTHREAD_MUTEX_INITIALIZER, 1, 0};
    return run(&j, n_threads);
}

/* Pass 2: bases. off[p] = start (bases) of pair p's region (query then
 * target, contiguous); every region must start at a multiple of 4 bases so
 * that threads never share a 2-bit byte. u8 / b2 must be zero-initialised
 * (b2 is OR-ed into). */
int gen_bases(const gen_cfg_t *cfg, const int64_t *off, uint8_t *u8, uint8_t *b2, int n_threads) {
    job_t j = {cfg, NULL, NULL, NULL, NULL, off, u8, b2, NULL, 0, PTHREAD_MUTEX_INITIALIZER, 2, 0};
    return run(&j, n_threads);
}

/* Pass 2 for global pair indices idx[0 .. cfg->n_pairs) (see gen_lengths_idx). */
int gen_bases_idx(const gen_cfg_t *cfg, const int64_t *idx, const int64_t *off, uint8_t *u8, uint8_t *b2,
                  int n_threads) {
    job_t j = {cfg, NULL, NULL, NULL, NULL, off, u8, b2, idx, 0, PTHREAD_MUTEX_INITIALIZER, 2, 0};
    return run(&j, n_threads);
}
