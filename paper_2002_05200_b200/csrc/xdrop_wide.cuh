// xdrop_wide.cuh — the unbounded escalation level: one CTA per task, the
// three antidiagonals (Fig. 1) in a per-CTA global scratch indexed by
// the query offset i, threads strided along the antidiagonal in segments of
// the block width (Alg. 2), block-wide max / argmax / band
// reductions per antidiagonal.
//
// This is the paper's own intra-sequence scheme, kept only as the exact
// fallback for tasks whose band outgrows the widest register window (1024
// diagonal slots): e.g. long unrelated reads at large X (c-amb-17). Values are
// absolute int32 with an explicit dead marker; a column outside the range
// visited on an antidiagonal is dead (it had no live predecessor).
//
// Per antidiagonal: each thread sweeps its cells, warps reduce with CREDUX
// (max value, then smallest i at that value; smallest / largest live i), lane
// 0 of every warp writes its partials to a parity-double-buffered shared slot,
// ONE __syncthreads, then every warp folds the 32 partials with one LDS per lane
// and CREDUX (no second barrier: the next antidiagonal writes the other
// parity's slots).
#pragma once

#include "xdrop_common.cuh"

namespace logan {

constexpr int WIDE_THREADS = 1024;
constexpr int SUBST_THREADS = 256;  // substitution-matrix path: narrower CTAs (bands ~X cells)
constexpr int SUBST_MAX_ALPHABET = 32;
constexpr int32_t WDEAD = INT32_MIN;

// Substitution score s(a_i, b_j) (eq. P:85): match / mismatch, or with SUB the
// entry of the caller's matrix (protein alignment P:381),
// staged in shared memory as a 32 x 32 int8 table (codes < alphabet <= 32).
template <bool SUB>
__device__ __forceinline__ int32_t subst_score(const Params &P, const int8_t *tab, uint32_t a, uint32_t b) {
    if (SUB) return (int32_t)tab[(a & 31u) * SUBST_MAX_ALPHABET + (b & 31u)];
    return a == b ? P.match : P.mismatch;
}

template <int FMT, int NT = WIDE_THREADS, bool SUB = false>
__global__ void __launch_bounds__(NT) k_wide(const Params P, const LevelIO io,
                                             int32_t *scratch, int64_t stride) {
    constexpr int NWARP = NT / 32;
    __shared__ int32_t s_v[2][32], s_i[2][32], s_f[2][32], s_l[2][32];
    __shared__ uint32_t s_task;
    __shared__ int8_t s_tab[SUB ? SUBST_MAX_ALPHABET * SUBST_MAX_ALPHABET : 4];
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    if (SUB) {
        for (int q = tid; q < SUBST_MAX_ALPHABET * SUBST_MAX_ALPHABET; q += NT) {
            const int a = q / SUBST_MAX_ALPHABET, b = q % SUBST_MAX_ALPHABET;
            s_tab[q] = (a < P.alphabet && b < P.alphabet) ? P.subst[a * P.alphabet + b] : (int8_t)0;
        }
        __syncthreads();
    }
    int32_t *V[3] = {scratch + (int64_t)blockIdx.x * 3 * stride,
                     scratch + (int64_t)blockIdx.x * 3 * stride + stride,
                     scratch + (int64_t)blockIdx.x * 3 * stride + 2 * stride};
    const uint32_t count = *io.count;
    for (;;) {
        if (tid == 0) {
            const uint32_t pos = atomicAdd(io.cursor, 1u);
            s_task = pos < count ? io.list[pos] : NO_TASK;
        }
        __syncthreads();
        const uint32_t task = s_task;
        __syncthreads();
        if (task == NO_TASK) return;
        const TaskDesc td = task_desc(P, task);
        const int32_t m = td.a.len, n = td.b.len;
        if ((int64_t)m + 2 > stride) {  // caller's max_ext_len bound was too small
            if (tid == 0) {
                TaskRes tr;
                tr.best = 0; tr.i = 0; tr.j = 0; tr.flags = 2; tr.cells = 0;
                io.tres[task] = tr;
            }
            continue;
        }

        // per-antidiagonal bookkeeping (uniform across the block), rotated
        // scalars for d-1 ("1") and d-2 ("2"); buffers rotate through V[]
        int32_t lo1 = 0, hi1 = 0, F1 = 0, L1 = 0;  // antidiagonal 0: the origin
        bool h1 = true;
        int32_t lo2 = 0, hi2 = -1, F2 = 0, L2 = 0;
        bool h2 = false;
        int32_t *V0 = V[1], *V1 = V[0], *V2 = V[2];
        if (tid == 0) V1[0] = 0;  // origin S(0,0) = 0
        int32_t best = 0, ai = 0, aj = 0;
        int32_t li = 0, ld = 0;  // compat: the origin unless a later antidiagonal has a live cell
        uint64_t cells = 0;
        __syncthreads();

        for (int32_t d = 1;; ++d) {
            // band and visiting range (cells with a possibly live predecessor)
            int32_t lo = INT32_MAX, hi = INT32_MIN;
            if (h1) { lo = min(lo, F1); hi = max(hi, L1 + 1); }
            if (h2) { lo = min(lo, F2 + 1); hi = max(hi, L2 + 1); }
            if (d >= 2 && (h1 || h2)) {
                const int32_t blo = max(lo, max(1, d - n)), bhi = min(hi, min(m, d - 1));
                if (bhi >= blo) cells += (uint64_t)(bhi - blo + 1);
            }
            const int32_t vlo = max(lo, max(0, d - n)), vhi = min(hi, min(m, d));
            const int32_t thr = best - P.xdrop;
            int32_t bv = INT32_MIN, bi = INT32_MAX, lf = INT32_MAX, ll = INT32_MIN;
            for (int32_t i = vlo + tid; i <= vhi; i += NT) {
                const int32_t j = d - i;
                bool have = false;
                int32_t v = 0;
                if (i >= 1 && j >= 1 && h2 && i - 1 >= lo2 && i - 1 <= hi2) {
                    const int32_t p = V2[i - 1];
                    if (p != WDEAD) {
                        const uint32_t a = pool_base<FMT>(P, td.a.base + (int64_t)td.a.dir * (i - 1));
                        const uint32_t b = pool_base<FMT>(P, td.b.base + (int64_t)td.b.dir * (j - 1));
                        v = p + subst_score<SUB>(P, s_tab, a, b);
                        have = true;
                    }
                }
                if (j >= 1 && i >= lo1 && i <= hi1) {
                    const int32_t p = V1[i];
                    if (p != WDEAD) { v = have ? max(v, p + P.gap) : p + P.gap; have = true; }
                }
                if (i >= 1 && i - 1 >= lo1 && i - 1 <= hi1) {
                    const int32_t p = V1[i - 1];
                    if (p != WDEAD) { v = have ? max(v, p + P.gap) : p + P.gap; have = true; }
                }
                // drop iff S < best - X; SeqAn-compat (reading c-amb-24): boundary
                // cells (i = 0 or j = 0) on d >= 2 need S > best - X
                const bool live = have && ((P.compat && d >= 2 && (i == 0 || j == 0)) ? v > thr : v >= thr);
                V0[i] = live ? v : WDEAD;
                if (live) {
                    lf = min(lf, i);
                    ll = max(ll, i);
                    if (v > bv) { bv = v; bi = i; }  // ascending i: the first max is kept
                }
            }
            // warp reductions: max value, then the smallest i holding it
            const int32_t wv = __reduce_max_sync(0xffffffffu, bv);
            const int32_t wi = __reduce_min_sync(0xffffffffu, bv == wv ? bi : INT32_MAX);
            const int32_t wf = __reduce_min_sync(0xffffffffu, lf);
            const int32_t wl = __reduce_max_sync(0xffffffffu, ll);
            const int par = d & 1;
            if (lane == 0) { s_v[par][wid] = wv; s_i[par][wid] = wi; s_f[par][wid] = wf; s_l[par][wid] = wl; }
            __syncthreads();  // also orders the V0 writes before the next antidiagonal
            // every warp folds the 32 partials the same way: lane q reads warp
            // q's slot (one LDS each) and CREDUX combines them
            const bool q_ok = lane < NWARP;
            const int32_t qv = q_ok ? s_v[par][lane] : INT32_MIN, qi = q_ok ? s_i[par][lane] : INT32_MAX;
            const int32_t gv = __reduce_max_sync(0xffffffffu, qv);
            const int32_t gi = __reduce_min_sync(0xffffffffu, qv == gv ? qi : INT32_MAX);
            const int32_t gf = __reduce_min_sync(0xffffffffu, q_ok ? s_f[par][lane] : INT32_MAX);
            const int32_t gl = __reduce_max_sync(0xffffffffu, q_ok ? s_l[par][lane] : INT32_MIN);
            const bool h0 = (gf != INT32_MAX);
            if (h0 && gv > best) { best = gv; ai = gi; aj = d - gi; }  // P:178, strict increase
            if (h0) { li = gi; ld = d; }  // compat (c-amb-25): the last live antidiagonal's best cell
            if (h0 && P.zdrop >= 0) {  // Z-drop stop (c-amb-19)
                const int32_t off = abs((gi - ai) - ((d - gi) - aj));
                if (best - gv > P.zdrop - P.gap * off) break;
            }
            if (!h0 && !h1) break;  // P:186, c-amb-7
            // rotate: d becomes "1", d-1 becomes "2"
            lo2 = lo1; hi2 = hi1; F2 = F1; L2 = L1; h2 = h1;
            lo1 = vlo; hi1 = vhi; F1 = gf; L1 = gl; h1 = h0;
            int32_t *t = V2; V2 = V1; V1 = V0; V0 = t;
        }
        if (tid == 0) {
            TaskRes tr;
            tr.best = best;
            tr.i = P.compat ? li : ai;  // compat: the "longest extension" cell (c-amb-25)
            tr.j = P.compat ? ld - li : aj;
            tr.flags = 0;
            tr.cells = cells;
            io.tres[task] = tr;
            if (io.stats) {
                atomicAdd((unsigned long long *)&io.stats->tasks_started[io.level], 1ull);
                atomicAdd((unsigned long long *)&io.stats->tasks_finished[io.level], 1ull);  // restarted here
                atomicAdd((unsigned long long *)&io.stats->cells_per_level[io.level], (unsigned long long)cells);
                atomicAdd((unsigned long long *)&io.stats->cells_total, (unsigned long long)cells);
            }
        }
        __syncthreads();  // both parities' slots are reused by the next task
    }
}

}  // namespace logan
