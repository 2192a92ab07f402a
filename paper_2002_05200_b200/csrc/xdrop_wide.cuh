// xdrop_wide.cuh — the unbounded escalation level: one CTA per task, the
// three antidiagonals (Fig. 1) in a per-CTA global scratch indexed by
// the query offset i, threads strided along the antidiagonal in segments of
// the block width (Alg. 2), block-wide max / argmax / band
// reductions per antidiagonal.
//
// This is the paper's own intra-sequence scheme, kept only as the exact
// fallback for tasks whose band outgrows the widest register window (1024
// diagonal slots): e.g. unrelated reads at large X (c-amb-17). Values are
// absolute int32 with an explicit dead marker; a column outside the range
// visited on an antidiagonal is dead (it had no live predecessor).
#pragma once

#include "xdrop_common.cuh"

namespace logan {

constexpr int WIDE_THREADS = 256;
constexpr int32_t WDEAD = INT32_MIN;

__device__ __forceinline__ unsigned long long wide_key(int32_t v, int32_t i) {
    // max over keys = max value, then smallest i
    return ((unsigned long long)((uint32_t)v ^ 0x80000000u) << 32) | (uint32_t)(~(uint32_t)i);
}

template <int FMT>
__global__ void __launch_bounds__(WIDE_THREADS) k_wide(const Params P, const LevelIO io,
                                                       int32_t *scratch, int64_t stride) {
    __shared__ unsigned long long s_key[WIDE_THREADS / 32];
    __shared__ int32_t s_f[WIDE_THREADS / 32], s_l[WIDE_THREADS / 32];
    __shared__ uint32_t s_task;
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
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

        // per-antidiagonal bookkeeping (uniform across the block)
        int32_t vis_lo[3] = {0, 0, 0}, vis_hi[3] = {-1, -1, -1};
        int32_t F[3] = {0, 0, 0}, L[3] = {0, 0, 0};
        bool has[3] = {false, false, false};
        if (tid == 0) V[0][0] = 0;  // origin S(0,0) = 0
        vis_lo[0] = vis_hi[0] = 0;
        F[0] = L[0] = 0;
        has[0] = true;
        int32_t best = 0, ai = 0, aj = 0;
        uint64_t cells = 0;
        __syncthreads();

        for (int32_t d = 1;; ++d) {
            const int c = d % 3, c1 = (d + 2) % 3, c2 = (d + 1) % 3;
            const bool h1 = has[c1], h2 = (d >= 2) && has[c2];
            // band and visiting range (cells with a possibly live predecessor)
            int32_t lo = INT32_MAX, hi = INT32_MIN;
            if (h1) { lo = min(lo, F[c1]); hi = max(hi, L[c1] + 1); }
            if (h2) { lo = min(lo, F[c2] + 1); hi = max(hi, L[c2] + 1); }
            if (d >= 2 && (h1 || h2)) {
                const int32_t blo = max(lo, max(1, d - n)), bhi = min(hi, min(m, d - 1));
                if (bhi >= blo) cells += (uint64_t)(bhi - blo + 1);
            }
            const int32_t vlo = max(lo, max(0, d - n)), vhi = min(hi, min(m, d));
            const int32_t thr = best - P.xdrop;
            unsigned long long kbest = 0;
            int32_t lf = INT32_MAX, ll = INT32_MIN;
            const int32_t *V1 = V[c1], *V2 = V[c2];
            int32_t *V0 = V[c];
            const int32_t lo1 = vis_lo[c1], hi1 = vis_hi[c1], lo2 = vis_lo[c2], hi2 = vis_hi[c2];
            for (int32_t i = vlo + tid; i <= vhi; i += WIDE_THREADS) {
                const int32_t j = d - i;
                bool have = false;
                int32_t v = 0;
                if (i >= 1 && j >= 1 && d >= 2 && i - 1 >= lo2 && i - 1 <= hi2) {
                    const int32_t p = V2[i - 1];
                    if (p != WDEAD) {
                        const uint32_t a = seq_at<FMT>(P, td.a, i, 0xffffffffu);
                        const uint32_t b = seq_at<FMT>(P, td.b, j, 0xfffffffeu);
                        v = p + (a == b ? P.match : P.mismatch);
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
                const bool live = have && v >= thr;  // drop iff S < best - X
                V0[i] = live ? v : WDEAD;
                if (live) {
                    lf = min(lf, i);
                    ll = max(ll, i);
                    const unsigned long long key = wide_key(v, i);
                    kbest = key > kbest ? key : kbest;
                }
            }
            // block reductions
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long ok = __shfl_xor_sync(0xffffffffu, kbest, o);
                kbest = ok > kbest ? ok : kbest;
            }
            lf = __reduce_min_sync(0xffffffffu, lf);
            ll = __reduce_max_sync(0xffffffffu, ll);
            if (lane == 0) { s_key[wid] = kbest; s_f[wid] = lf; s_l[wid] = ll; }
            __syncthreads();  // also orders the V0 writes before the next antidiagonal
            kbest = 0;
            lf = INT32_MAX;
            ll = INT32_MIN;
#pragma unroll
            for (int q = 0; q < WIDE_THREADS / 32; ++q) {
                kbest = s_key[q] > kbest ? s_key[q] : kbest;
                lf = min(lf, s_f[q]);
                ll = max(ll, s_l[q]);
            }
            __syncthreads();
            vis_lo[c] = vlo;
            vis_hi[c] = vhi;
            has[c] = (lf != INT32_MAX);
            F[c] = lf;
            L[c] = ll;
            if (kbest != 0) {
                const int32_t v = (int32_t)((uint32_t)(kbest >> 32) ^ 0x80000000u);
                const int32_t i = (int32_t)(~(uint32_t)kbest);
                if (v > best) { best = v; ai = i; aj = d - i; }  // P:178, strict increase
            }
            if (!has[c] && !has[c1]) break;  // P:186, c-amb-7
        }
        if (tid == 0) {
            TaskRes tr;
            tr.best = best;
            tr.i = ai;
            tr.j = aj;
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
    }
}

}  // namespace logan
