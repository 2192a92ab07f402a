// logan_impl.cuh — device pipeline of the B200 X-drop library (kernels, level
// table, run_batch<FMT>). Included by logan_xdrop.cu (the C ABI) and by one
// translation unit per format (logan_fmt*.cu), which instantiate run_batch for
// that format only, so the build compiles the formats in parallel.
#pragma once
#include <cstdio>
#include <cstring>
#include "logan_xdrop.h"
#include "xdrop_common.cuh"
#include "xdrop_band.cuh"
#include "xdrop_wide.cuh"
#include "xdrop_window.cuh"
#include "xdrop_window16.cuh"

namespace logan {

constexpr int NBUCKET = 2048;
constexpr int NLEVEL = 8;  // 6 window levels + the band level + the CTA level
constexpr int BAND_LEVEL = 6, WIDE_LEVEL = 7;
constexpr int SETUP_THREADS = 256;
constexpr int32_t XDROP_MAX = 1 << 28;   // ABI limit on X and Z
constexpr int32_t WINDOW_XMAX = 1 << 19; // register windows: (X + 2*127) * KEYMUL < 2^31

__device__ __forceinline__ uint32_t cost_bucket(uint32_t c) {
    // monotone log-linear bucket: 32 octaves x 64 sub-buckets (c >= 1)
    const uint32_t e = 31u - __clz(c);
    const uint32_t mant = e >= 6 ? (c >> (e - 6)) & 63u : (c << (6 - e)) & 63u;
    return e * 64u + mant;
}

// Workspace layout (each region 256-byte aligned).
// First-level window: one lane per task x w0 slots, w0 in {20, 24, 28, 32}
// chosen at run time from X and the read lengths (auto_first_slots), or forced
// by options.first_slots.
constexpr int NWIDTH = 6;  // register-window widths w0, 64, 128, 256, 512, 1024
static const int kWidth[NWIDTH] = {32, 64, 128, 256, 512, 1024};  // [0]: the largest w0 (pool sizing)

struct Layout {
    size_t tres, tbucket, queue, listA, listB, recsA, recsB, hist, cursor_b, counters, wide, total;
    size_t pool[NWIDTH];         // hand-over records written by window level w
    uint32_t pool_cap[NWIDTH];
    int64_t ntask, wide_stride;
};

constexpr int WIDE_CTAS = 296;  // 2 per SM on B200
constexpr int NCTR = 64;
constexpr int CTR_OUT = 16, CTR_FILL = 32, CTR_DONE = 48;
constexpr int CTR_BAND2_CURSOR = 10, CTR_BAND2_OUT = 25;  // the band level's second stage

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static Layout make_layout(int64_t n_pairs, int64_t max_ext_len) {
    Layout L{};
    const int64_t nt = 2 * n_pairs;
    L.ntask = nt;
    size_t o = 0;
    L.tres = o;     o += align256(sizeof(TaskRes) * (size_t)nt);
    L.tbucket = o;  o += align256(sizeof(uint16_t) * (size_t)nt);
    L.queue = o;    o += align256(sizeof(uint32_t) * (size_t)nt);
    L.listA = o;    o += align256(sizeof(uint32_t) * (size_t)nt);
    L.listB = o;    o += align256(sizeof(uint32_t) * (size_t)nt);
    L.recsA = o;    o += align256(sizeof(uint32_t) * (size_t)nt);
    L.recsB = o;    o += align256(sizeof(uint32_t) * (size_t)nt);
    for (int w = 0; w < NWIDTH; ++w) {
        // at most 128 MiB of records per level; tasks beyond that restart
        const int64_t rec_bytes = (int64_t)sizeof(int32_t) * rec_ints(kWidth[w]);
        int64_t cap = ((int64_t)128 << 20) / rec_bytes;
        if (cap > nt) cap = nt;
        L.pool_cap[w] = (uint32_t)cap;
        L.pool[w] = o;
        o += align256((size_t)(rec_bytes * cap));
    }
    L.hist = o;     o += align256(sizeof(uint32_t) * NBUCKET);
    L.cursor_b = o; o += align256(sizeof(uint32_t) * NBUCKET);
    // counters: [0] queue count, [1 + lv] level cursors, [16 + lv] out counts,
    // [32 + lv] record pool fill, [48] producer groups done (helpers)
    L.counters = o; o += align256(sizeof(uint32_t) * NCTR);
    L.wide_stride = max_ext_len + 2;
    L.wide = o;     o += align256(sizeof(int32_t) * 3 * (size_t)L.wide_stride * WIDE_CTAS);
    L.total = o;
    return L;
}

// ---------------------------------------------------------------------------
static __global__ void k_expand(const Params P, TaskRes *tres, uint16_t *tbucket, uint32_t *hist) {
    __shared__ uint32_t sh[NBUCKET];
    for (int b = threadIdx.x; b < NBUCKET; b += blockDim.x) sh[b] = 0;
    __syncthreads();
    uint32_t n_bad = 0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P.n_pairs;
         p += (int64_t)gridDim.x * blockDim.x) {
        const bool ok = pair_valid(P, p);
        n_bad += ok ? 0u : 1u;
#pragma unroll
        for (int side = 0; side < 2; ++side) {
            const uint32_t task = (uint32_t)(2 * p + side);
            int32_t m = 0, n = 0;
            if (ok) {
                const int32_t ql = P.q_len[p], tl = P.t_len[p], qs = P.q_seed[p], ts = P.t_seed[p];
                m = side == 0 ? qs : ql - qs - P.k;
                n = side == 0 ? ts : tl - ts - P.k;
            }
            uint16_t bk = 0xffff;  // not queued
            if (ok && m > 0 && n > 0) {
                bk = (uint16_t)cost_bucket((uint32_t)(m + n));
                atomicAdd(&sh[bk], 1u);
            } else {
                TaskRes tr;
                tr.best = 0; tr.i = 0; tr.j = 0; tr.flags = ok ? 0 : 1; tr.cells = 0;
                tres[task] = tr;  // empty extension (c-amb-13) or invalid pair
            }
            tbucket[task] = bk;
        }
    }
    if (P.stats && n_bad) atomicAdd((unsigned long long *)&P.stats->pairs_invalid, (unsigned long long)n_bad);
    if (P.stats && blockIdx.x == 0 && threadIdx.x == 0) {
        P.stats->first_level = P.info[0];
        P.stats->first_width = P.info[1];
        P.stats->first_shape = P.info[2];
        P.stats->first_helpers = P.info[3];
    }
    __syncthreads();
    for (int b = threadIdx.x; b < NBUCKET; b += blockDim.x)
        if (sh[b]) atomicAdd(&hist[b], sh[b]);
}

// descending exclusive scan of the histogram (largest costs first)
static __global__ void k_scan(const uint32_t *hist, uint32_t *cursor_b, uint32_t *qcount) {
    __shared__ uint32_t part[SETUP_THREADS];
    constexpr int PER = NBUCKET / SETUP_THREADS;
    const int t = threadIdx.x;
    // thread t owns buckets in descending order: positions [t*PER, (t+1)*PER) of the reversed array
    uint32_t loc[PER];
    uint32_t s = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        loc[q] = hist[NBUCKET - 1 - (t * PER + q)];
        s += loc[q];
    }
    part[t] = s;
    __syncthreads();
    for (int o = 1; o < SETUP_THREADS; o <<= 1) {
        const uint32_t v = t >= o ? part[t - o] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    uint32_t run = part[t] - s;  // exclusive
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        cursor_b[NBUCKET - 1 - (t * PER + q)] = run;
        run += loc[q];
    }
    if (t == SETUP_THREADS - 1) *qcount = part[t];
}

static __global__ void k_scatter(int64_t ntask, const uint16_t *tbucket, uint32_t *cursor_b, uint32_t *queue) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntask;
         t += (int64_t)gridDim.x * blockDim.x) {
        const uint16_t b = tbucket[t];
        if (b != 0xffff) {
            const uint32_t pos = atomicAdd(&cursor_b[b], 1u);
            queue[pos] = (uint32_t)t;
        }
    }
}

template <int FMT>
static __global__ void k_combine(const Params P, const TaskRes *tres, logan_result_t *out, uint64_t *cells) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P.n_pairs;
         p += (int64_t)gridDim.x * blockDim.x) {
        const TaskRes L = tres[2 * p], R = tres[2 * p + 1];
        logan_result_t r;
        if ((L.flags | R.flags) & 3) {  // invalid pair (flags 2, the CTA level's scratch guard, cannot occur:
                                         // pair_valid rejects extensions above the bound that sizes it)
            r = {INT32_MIN, -1, -1, -1, -1};
            if (cells) cells[p] = 0;
        } else {
            const int64_t qo = P.q_off[p], to = P.t_off[p];
            const int32_t qs = P.q_seed[p], ts = P.t_seed[p];
            int32_t seed = 0;  // ungapped seed score (c-amb-10)
            for (int32_t u = 0; u < P.k; ++u) {
                const uint32_t a = pool_base<FMT>(P, qo + qs + u), b = pool_base<FMT>(P, to + ts + u);
                if (P.subst) seed += ((a & 31u) < (uint32_t)P.alphabet && (b & 31u) < (uint32_t)P.alphabet)
                                         ? P.subst[(a & 31u) * P.alphabet + (b & 31u)] : 0;
                else seed += a == b ? P.match : P.mismatch;
            }
            r.score = seed + L.best + R.best;
            r.q_begin = qs - L.i;
            r.q_end = qs + P.k + R.i;
            r.t_begin = ts - L.j;
            r.t_end = ts + P.k + R.j;
            if (cells) cells[p] = L.cells + R.cells;
        }
        out[p] = r;
    }
}

// ---------------------------------------------------------------------------
// Level table: register windows of W = 32, 64, 128, 256, 1024 diagonal slots.
// Throughput shape: G = W/32 lanes x R = 32 slots (many tasks in flight).
// Latency shape: one warp per task, R = W/32 slots per lane (few tasks left:
// the step's critical path is short). Level 5 is the unbounded CTA path.
// Helper shape for the first level: the next width's throughput shape (many
// tasks per helper warp, default) or its latency shape (one warp per task);
// LOGAN_HELPER_WARPS warps (the last warp of as many blocks) are helpers.
#ifndef LOGAN_HELPER_THROUGHPUT
#define LOGAN_HELPER_THROUGHPUT 1
#endif
#ifndef LOGAN_HELPER_WARPS  // 24 since the helpers are packed (profiles/r02/ab_helper_warps*.txt: 96 -> 48 -> 24:
#define LOGAN_HELPER_WARPS 24  // C3 X = 50 +3%, the C3 3/8 share 9.97 -> 8.88 ms, C3 / C2 / C4 unchanged)
#endif
#if LOGAN_HELPER_THROUGHPUT
#define LOGAN_HSHAPE(W) ((W) / 32), 32
#else
#define LOGAN_HSHAPE(W) 32, ((W) / 32)
#endif
// helpers of the packed first window (A/B knob): 4 x 16 instead of 2 x 32 fits the
// kernel into 128 registers (4 blocks per SM with LOGAN_PK_MINB 4), but measured
// slower (C3 1309-1323 vs 1345 GCUPS, C2 1231 vs 1275: half the helper capacity
// leaves a level-2 tail, and 16 warps per SM do not raise the ALU-bound rate)
#ifndef LOGAN_L1_G2_WARPS  // level 1 below this many one-lane warps per SM: two lanes per task
#define LOGAN_L1_G2_WARPS 0
#endif
#ifndef LOGAN_PK_HSHAPE
#define LOGAN_PK_HSHAPE LOGAN_HSHAPE(64)
#endif

template <int G, int R, int FMT, int HG, int HR, int PK = 0>
static cudaError_t launch_win(const Params &P, const LevelIO &io_in, const LevelIO &hio, int sms, cudaStream_t s) {
    constexpr int S1 = Window<G, R, FMT>::SB_STRIDE;
    constexpr int S2 = HR > 0 ? Window<(HG > 0 ? HG : 32), (HR > 0 ? HR : 1), FMT>::SB_STRIDE : 0;
    const size_t smem = 128 * sizeof(int32_t) * (S1 > S2 ? S1 : S2) + (fmt_base(FMT) == FMT_U8S ? SUBST_TAB_BYTES : 0);
    auto kern = k_window<G, R, FMT, HG, HR, PK>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    const int grid = sms * occ;
    LevelIO io = io_in;
    if (HR > 0) {
        io.helpers = grid < LOGAN_HELPER_WARPS ? grid : LOGAN_HELPER_WARPS;
        io.workers = (uint32_t)((grid * 128 - io.helpers * 32) / G);
    } else {
        io.helpers = 0;
    }
    kern<<<grid, 128, smem, s>>>(P, io, hio);
    return cudaGetLastError();
}

// the packed first window (2-bit pools, X <= 16000); PK 2 = match - mismatch = 2
template <int FMT, int PK>
static cudaError_t launch_first_pk(int w0, bool helpers, bool g2, const Params &P, const LevelIO &io,
                                   const LevelIO &hio, int sms, cudaStream_t s) {
    // few tasks: the 32-slot window on two lanes per task (2 x 16 slots)
    if (g2 && w0 == 32)
        return helpers ? launch_win<2, 16, FMT, LOGAN_PK_HSHAPE, PK>(P, io, hio, sms, s)
                       : launch_win<2, 16, FMT, 0, 0, PK>(P, io, hio, sms, s);
    switch (w0) {
        case 16: return helpers ? launch_win<1, 16, FMT, LOGAN_PK_HSHAPE, PK>(P, io, hio, sms, s)
                                : launch_win<1, 16, FMT, 0, 0, PK>(P, io, hio, sms, s);
        case 20: return helpers ? launch_win<1, 20, FMT, LOGAN_PK_HSHAPE, PK>(P, io, hio, sms, s)
                                : launch_win<1, 20, FMT, 0, 0, PK>(P, io, hio, sms, s);
        case 24: return helpers ? launch_win<1, 24, FMT, LOGAN_PK_HSHAPE, PK>(P, io, hio, sms, s)
                                : launch_win<1, 24, FMT, 0, 0, PK>(P, io, hio, sms, s);
        case 28: return helpers ? launch_win<1, 28, FMT, LOGAN_PK_HSHAPE, PK>(P, io, hio, sms, s)
                                : launch_win<1, 28, FMT, 0, 0, PK>(P, io, hio, sms, s);
        default: return helpers ? launch_win<1, 32, FMT, LOGAN_PK_HSHAPE, PK>(P, io, hio, sms, s)
                                : launch_win<1, 32, FMT, 0, 0, PK>(P, io, hio, sms, s);
    }
}

// wi = width index; latency = run the latency shape; helpers = first level with
// in-kernel escalation helpers running the next width
template <int FMT>
static cudaError_t launch_first(int w0, bool helpers, bool g2, const Params &P, const LevelIO &io,
                                const LevelIO &hio, int sms, cudaStream_t s) {
    // 2-bit pools (no Z-drop) at X <= 16000: the packed int16 window (xdrop_window16.cuh)
    if constexpr (FMT == LOGAN_SEQ_2BIT) {
        if (P.xdrop <= PACK_XMAX && !P.nopack) {
#ifndef LOGAN_NO_M2
            if (P.match - P.mismatch == 2) return launch_first_pk<FMT, 2>(w0, helpers, g2, P, io, hio, sms, s);
#endif
            return launch_first_pk<FMT, 1>(w0, helpers, g2, P, io, hio, sms, s);
        }
    }
    switch (w0) {
        case 16: return helpers ? launch_win<1, 16, FMT, LOGAN_HSHAPE(64)>(P, io, hio, sms, s)
                                : launch_win<1, 16, FMT, 0, 0>(P, io, hio, sms, s);
        case 20: return helpers ? launch_win<1, 20, FMT, LOGAN_HSHAPE(64)>(P, io, hio, sms, s)
                                : launch_win<1, 20, FMT, 0, 0>(P, io, hio, sms, s);
        case 24: return helpers ? launch_win<1, 24, FMT, LOGAN_HSHAPE(64)>(P, io, hio, sms, s)
                                : launch_win<1, 24, FMT, 0, 0>(P, io, hio, sms, s);
        case 28: return helpers ? launch_win<1, 28, FMT, LOGAN_HSHAPE(64)>(P, io, hio, sms, s)
                                : launch_win<1, 28, FMT, 0, 0>(P, io, hio, sms, s);
        default: return helpers ? launch_win<1, 32, FMT, LOGAN_HSHAPE(64)>(P, io, hio, sms, s)
                                : launch_win<1, 32, FMT, 0, 0>(P, io, hio, sms, s);
    }
}

// the packed windows of levels 2-6 (2-bit pools, X <= 16000); PK 2 = match - mismatch = 2;
// cudaErrorNotSupported = no packed shape (the int32 one runs)
template <int FMT, int PK>
static cudaError_t launch_width_pk(int wi, bool latency, bool helpers, const Params &P, const LevelIO &io,
                                   const LevelIO &hio, int sms, cudaStream_t s, int w5) {
    if (helpers && !latency) switch (wi) {
        case 1: return launch_win<2, 32, FMT, LOGAN_HSHAPE(128), PK>(P, io, hio, sms, s);
        case 2: return launch_win<4, 32, FMT, LOGAN_HSHAPE(256), PK>(P, io, hio, sms, s);
        case 3: return launch_win<8, 32, FMT, LOGAN_HSHAPE(512), PK>(P, io, hio, sms, s);
        case 4:
            if (w5 == 640) return launch_win<16, 32, FMT, 32, 20, PK>(P, io, hio, sms, s);
            if (w5 == 768) return launch_win<16, 32, FMT, 32, 24, PK>(P, io, hio, sms, s);
            if (w5 == 896) return launch_win<16, 32, FMT, 32, 28, PK>(P, io, hio, sms, s);
            return launch_win<16, 32, FMT, 32, 32, PK>(P, io, hio, sms, s);
        default: break;
    }
    if (wi == 5) {
        if (w5 == 640) return launch_win<32, 20, FMT, 0, 0, PK>(P, io, hio, sms, s);
        if (w5 == 768) return launch_win<32, 24, FMT, 0, 0, PK>(P, io, hio, sms, s);
        if (w5 == 896) return launch_win<32, 28, FMT, 0, 0, PK>(P, io, hio, sms, s);
        return launch_win<32, 32, FMT, 0, 0, PK>(P, io, hio, sms, s);
    }
    switch (wi * 2 + (latency ? 1 : 0)) {
        case 2: return launch_win<2, 32, FMT, 0, 0, PK>(P, io, hio, sms, s);
        case 4: return launch_win<4, 32, FMT, 0, 0, PK>(P, io, hio, sms, s);
        case 6: return launch_win<8, 32, FMT, 0, 0, PK>(P, io, hio, sms, s);
        case 8: return launch_win<16, 32, FMT, 0, 0, PK>(P, io, hio, sms, s);
        case 5: return launch_win<32, 4, FMT, 0, 0, PK>(P, io, hio, sms, s);   // W = 128, one warp
        case 7: return launch_win<32, 8, FMT, 0, 0, PK>(P, io, hio, sms, s);   // W = 256, one warp
        case 9: return launch_win<32, 16, FMT, 0, 0, PK>(P, io, hio, sms, s);
        default: break;  // W = 64 on one warp (2 slots per lane): int32
    }
    return cudaErrorNotSupported;
}

template <int FMT>
static cudaError_t launch_width(int wi, bool latency, bool helpers, const Params &P, const LevelIO &io,
                                const LevelIO &hio, int sms, cudaStream_t s, int w0, int w5, bool g2 = false) {
    if (wi == 0 && !(latency && w0 == 32)) return launch_first<FMT>(w0, helpers && !latency, g2, P, io, hio, sms, s);
    // 2-bit pools (no Z-drop) at X <= 16000: the packed int16 windows for the
    // throughput shapes (G x 32 slots) and the one-warp shapes of W >= 128 (4 or more slots per lane)
    if constexpr (FMT == LOGAN_SEQ_2BIT) {
        if (P.xdrop <= PACK_XMAX && !P.nopack) {
#ifndef LOGAN_NO_M2
            if (P.match - P.mismatch == 2) {
                const cudaError_t e = launch_width_pk<FMT, 2>(wi, latency, helpers, P, io, hio, sms, s, w5);
                if (e != cudaErrorNotSupported) return e;
            } else
#endif
            {
                const cudaError_t e = launch_width_pk<FMT, 1>(wi, latency, helpers, P, io, hio, sms, s, w5);
                if (e != cudaErrorNotSupported) return e;
            }
        }
    }
    constexpr bool HELP = true;
    if (HELP && helpers && !latency) {
        if constexpr (HELP) switch (wi) {
            case 1: return launch_win<2, 32, FMT, LOGAN_HSHAPE(128)>(P, io, hio, sms, s);
            case 2: return launch_win<4, 32, FMT, LOGAN_HSHAPE(256)>(P, io, hio, sms, s);
            case 3: return launch_win<8, 32, FMT, LOGAN_HSHAPE(512)>(P, io, hio, sms, s);
            case 4:
                if (w5 == 640) return launch_win<16, 32, FMT, 32, 20>(P, io, hio, sms, s);
                if (w5 == 768) return launch_win<16, 32, FMT, 32, 24>(P, io, hio, sms, s);
                if (w5 == 896) return launch_win<16, 32, FMT, 32, 28>(P, io, hio, sms, s);
                return launch_win<16, 32, FMT, 32, 32>(P, io, hio, sms, s);
            default: break;
        }
    }
    if (wi == 5) {  // the top window: one warp per task, R = w5 / 32 slots per lane
        if (w5 == 640) return launch_win<32, 20, FMT, 0, 0>(P, io, hio, sms, s);
        if (w5 == 768) return launch_win<32, 24, FMT, 0, 0>(P, io, hio, sms, s);
        if (w5 == 896) return launch_win<32, 28, FMT, 0, 0>(P, io, hio, sms, s);
    }
    switch (wi * 2 + (latency ? 1 : 0)) {
        case 1: return launch_win<32, 1, FMT, 0, 0>(P, io, hio, sms, s);
        case 2: return launch_win<2, 32, FMT, 0, 0>(P, io, hio, sms, s);
        case 3: return launch_win<32, 2, FMT, 0, 0>(P, io, hio, sms, s);
        case 4: return launch_win<4, 32, FMT, 0, 0>(P, io, hio, sms, s);
        case 5: return launch_win<32, 4, FMT, 0, 0>(P, io, hio, sms, s);
        case 6: return launch_win<8, 32, FMT, 0, 0>(P, io, hio, sms, s);
        case 7: return launch_win<32, 8, FMT, 0, 0>(P, io, hio, sms, s);
        case 8: return launch_win<16, 32, FMT, 0, 0>(P, io, hio, sms, s);
        case 9: return launch_win<32, 16, FMT, 0, 0>(P, io, hio, sms, s);
        case 10:
        case 11: return launch_win<32, 32, FMT, 0, 0>(P, io, hio, sms, s);
        default: return cudaErrorInvalidValue;
    }
}

static int auto_first_level(int32_t xdrop) {
    // the band of true pairs is about X + a few slots wide
    if (xdrop <= 20) return 0;   // W = w0 (auto_first_slots)
    if (xdrop <= 50) return 1;   // W = 64
    if (xdrop <= 110) return 2;  // W = 128
    if (xdrop <= 230) return 3;  // W = 256
    if (xdrop <= 480) return 4;  // W = 512
    if (xdrop <= 1000) return 5; // W = 1024
    if (xdrop <= BAND_XMAX) return BAND_LEVEL;  // the band follows the alignment's width
    return WIDE_LEVEL;           // unbounded CTA level
}

// Width of the top window level (one warp per task): 640, 768 or 896 slots when
// X starts tasks there with a band of about X + 8 slots (X in (480, 820]), so
// the window is not half empty; 1024 otherwise (X near 1000, or bands that
// escalated from narrower windows, e.g. spurious pairs at small X).
static int auto_top_width(int32_t xdrop) {
    if (xdrop <= 480) return 1024;
    if (xdrop <= 560) return 640;
    if (xdrop <= 680) return 768;
    if (xdrop <= 820) return 896;
    return 1024;
}

// Slots of the first window: the band of true pairs is about X + 8 slots wide at
// its widest, and long reads drift more between re-centrings.
// Measured on C6 / C3 (profiles/r01_ab_first_slots_small_x.txt): X = 5: 16 slots
// 617 GCUPS vs 20: 555; X = 8: 20 754 vs 16: 614 (2% of tasks overflow); X = 10:
// 20 ~ 24 on 2.5-7.5 kb reads, 24 +10% on 10 kb reads; X = 12: 24 881 vs 20: 730;
// X = 14, 16: 24 best; X = 18, 20: 28 best on 2.5-7.5 kb reads (C6 X = 20: 1168 vs
// 32: 1109), 32 on 10 kb reads (profiles/r01_ab_first_slots_mid_x.txt). Round 2,
// packed window (profiles/r02/ab_slots_v10.txt, ab_slots_v12.txt): X = 10 takes 24
// slots (C3 998 vs 32: 948; C2 920 vs 20: 870), X in (10, 20] 32 slots on every read
// length (C3 X = 16: 1370 vs 28: 1255, 24: 766; C2 X = 20: 1391 vs 28: 1334).
static int auto_first_slots(int32_t xdrop, int64_t max_ext) {
    (void)max_ext;
    if (xdrop <= 5) return 16;
    if (xdrop <= 10) return 24;
    return 32;
}

// one persistent launch of the band level in configuration C (xdrop_band.cuh)
template <int FMT, class C>
static cudaError_t launch_band(const Params &P, const LevelIO &io, int sms, cudaStream_t s) {
    const int smem = (int)BandSmem<FMT, C>::BYTES;
    cudaError_t e = cudaFuncSetAttribute(k_band<FMT, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_band<FMT, C>, C::NT, smem);
    if (e != cudaSuccess) return e;
    k_band<FMT, C><<<sms * (per_sm > 0 ? per_sm : 1), C::NT, smem, s>>>(P, io);
    return cudaGetLastError();
}

template <int FMT>
int run_batch(const Params &P, const logan_options_t *opt, bool wide_only, logan_result_t *out, uint64_t *cells,
                     logan_stats_t *stats, uint8_t *ws, const Layout &L, cudaStream_t s) {
    TaskRes *tres = (TaskRes *)(ws + L.tres);
    uint16_t *tbucket = (uint16_t *)(ws + L.tbucket);
    uint32_t *queue = (uint32_t *)(ws + L.queue);
    uint32_t *lists[2] = {(uint32_t *)(ws + L.listA), (uint32_t *)(ws + L.listB)};
    uint32_t *hist = (uint32_t *)(ws + L.hist);
    uint32_t *cursor_b = (uint32_t *)(ws + L.cursor_b);
    uint32_t *ctr = (uint32_t *)(ws + L.counters);
    int32_t *wide = (int32_t *)(ws + L.wide);

    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess) return LOGAN_ECUDA;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return LOGAN_ECUDA;

    if (cudaMemsetAsync(hist, 0, sizeof(uint32_t) * NBUCKET, s) != cudaSuccess) return LOGAN_ECUDA;
    if (cudaMemsetAsync(ctr, 0, sizeof(uint32_t) * NCTR, s) != cudaSuccess) return LOGAN_ECUDA;
    if (stats && cudaMemsetAsync(stats, 0, sizeof(logan_stats_t), s) != cudaSuccess) return LOGAN_ECUDA;

    cudaEvent_t const *ev = (opt && opt->timing_events) ? (cudaEvent_t const *)opt->timing_events : nullptr;
    auto mark = [&](int stage, int which) -> bool {
        return !ev || cudaEventRecord(ev[2 * stage + which], s) == cudaSuccess;
    };
    // level choice from the expected band width: about X slots under +1/-1/-1;
    // with a substitution matrix about X / |gap| (moving one slot off the
    // alignment's diagonal costs two gaps against at most X of slack)
    const int32_t xband = fmt_base(FMT) == FMT_U8S ? (P.xdrop + (-P.gap) - 1) / (-P.gap) : P.xdrop;
    int first = (opt && opt->first_level > 0) ? opt->first_level - 1 : auto_first_level(xband);
    if (wide_only) first = WIDE_LEVEL;  // X' > 2^19: beyond the windows' key range (header)
    // no band level for matrices or Z-drop: those tasks go on to the CTA level
    constexpr bool no_band = fmt_base(FMT) == FMT_U8S || fmt_z(FMT);
    if (no_band && first == BAND_LEVEL) first = WIDE_LEVEL;
    if (first < 0 || first > NLEVEL - 1) return LOGAN_EINVAL;
    uint32_t *recs[2] = {(uint32_t *)(ws + L.recsA), (uint32_t *)(ws + L.recsB)};
    // flags bit 0 at level 1: the 32-slot window, the only one with a latency shape
    const int w0 = (opt && opt->first_slots > 0) ? opt->first_slots
                   : ((opt && (opt->flags & 1)) ? 32 : auto_first_slots(xband, P.max_ext));
    const int w5 = auto_top_width(xband);
    auto width_of = [&](int lv) { return lv == 0 ? w0 : (lv == NWIDTH - 1 ? w5 : kWidth[lv]); };
    const uint32_t *in_list = queue;
    const uint32_t *in_recs = nullptr;
    const int32_t *rec_in = nullptr;
    int64_t rec_in_stride = 0;
    const uint32_t *in_count = &ctr[0];
    int out_sel = 0;
    // below this many tasks a level runs in its latency shape (one warp per task)
    const uint32_t latency_below = (uint32_t)sms * 16u;
    // the IO of window level lv, given its input list / records
    auto level_io = [&](int lv, const uint32_t *lst, const uint32_t *cnt, const uint32_t *irecs,
                        const int32_t *rin, int64_t rin_stride, int osel) {
        LevelIO io{};
        io.list = lst;
        io.count = cnt;
        io.cursor = &ctr[1 + lv];
        io.out_list = lists[osel];
        io.out_count = &ctr[CTR_OUT + lv];
        io.stats = stats;
        io.level = lv;
        io.tres = tres;
        io.in_recs = irecs;
        io.rec_in = rin;
        io.rec_in_stride = rin_stride;
        io.handover = opt ? opt->handover : 0;
        io.min_count = 0;
        io.max_count = 0xffffffffu;
        if (lv < NWIDTH) {
            io.out_recs = recs[osel];
            io.rec_out = (int32_t *)(ws + L.pool[lv]);
            io.rec_out_stride = rec_ints(width_of(lv));
            io.rec_out_cap = L.pool_cap[lv];
            io.rec_out_count = &ctr[CTR_FILL + lv];
        }
        return io;
    };
    // Few tasks (e.g. long reads spread over many GPUs): the throughput shape
    // would leave SMs with too few warps to hide the per-antidiagonal latency,
    // so the first level runs one warp per task instead (measured on C5 with
    // 2,500 pairs: 260 vs 158 GCUPS at 4.2 throughput-shape warps per SM; C3 at
    // X = 50 with 12,500 pairs, 10.6 warps per SM, prefers the throughput shape:
    // 487 vs 300 GCUPS, profiles/r01_ab_few_tasks.txt).
    const int64_t groups_needed = L.ntask * (first < NWIDTH ? width_of(first) / 32 : 1) / 32;  // warps
    // Level 1 (one lane per task) keeps its throughput shape down to 2 warps per SM;
    // its latency shape exists for the 32-slot window only (C3, X = 20: 3,000 pairs,
    // 1.3 warps/SM: 128 vs 95 GCUPS for latency; 6,250 pairs: 171 vs 121 for
    // throughput; profiles/r01_ab_l1_latency.txt).
    const bool few_tasks = (first > 0 && first < NWIDTH && groups_needed < (int64_t)sms * 8) ||
                           (first == 0 && w0 == 32 && groups_needed < (int64_t)sms * 2);
    const bool latency_first = (opt && (opt->flags & 1)) || (few_tasks && !(opt && (opt->flags & 8)));
    // Level 1 with few tasks but more than the latency shape's limit: the packed
    // 32-slot window on two lanes per task (twice the warps, half the dependent
    // chain per antidiagonal)
    const bool l1_g2 = first == 0 && w0 == 32 && !latency_first &&
                       groups_needed < (int64_t)sms * LOGAN_L1_G2_WARPS;
    // the first level's launch, recorded in stats (diagnostics: which kernel ran)
    Params Pe = P;
    if (stats) {
        const bool shape_lat = latency_first && !(first == 0 && w0 != 32);
        Pe.info[0] = (uint32_t)(first + 1);
        Pe.info[1] = first < NWIDTH ? (uint32_t)width_of(first) : 0u;
        Pe.info[2] = first < NWIDTH && shape_lat ? 1u : 0u;
        Pe.info[3] = first < NWIDTH - 1 && !latency_first ? 1u : 0u;
    }
    if (!mark(0, 0)) return LOGAN_ECUDA;
    const int64_t per_block = SETUP_THREADS;
    int grid = (int)((P.n_pairs + per_block - 1) / per_block);
    if (grid > sms * 8) grid = sms * 8;
    if (grid < 1) grid = 1;
    k_expand<<<grid, SETUP_THREADS, 0, s>>>(Pe, tres, tbucket, hist);
    k_scan<<<1, SETUP_THREADS, 0, s>>>(hist, cursor_b, &ctr[0]);
    int grid2 = (int)((L.ntask + per_block - 1) / per_block);
    if (grid2 > sms * 8) grid2 = sms * 8;
    if (grid2 < 1) grid2 = 1;
    k_scatter<<<grid2, SETUP_THREADS, 0, s>>>(L.ntask, tbucket, cursor_b, queue);
    if (cudaGetLastError() != cudaSuccess) return LOGAN_ECUDA;
    if (!mark(0, 1)) return LOGAN_ECUDA;

    bool band2 = false;  // the band level ran its second stage (its output list is the other one)
    for (int lv = first; lv < NLEVEL; ++lv) {
        // substitution matrices have no band level: tasks that outgrow the widest
        // window go straight on to the CTA level (which restarts them)
        if (no_band && lv == BAND_LEVEL) continue;
        LevelIO io = level_io(lv, in_list, in_count, in_recs, rec_in, rec_in_stride, out_sel);
        cudaError_t e = cudaSuccess;
        if (!mark(1 + lv, 0)) return LOGAN_ECUDA;
        if (lv < NWIDTH) {
            if (lv == first) {
                io.sms = sms;  // the first level's static first round (xdrop_window.cuh)
                const bool helpers = !latency_first && lv + 1 < NWIDTH;
                LevelIO hio{};
                if (helpers) {
                    // the next level's IO: it reads this level's hand-overs
                    hio = level_io(lv + 1, lists[out_sel], &ctr[CTR_OUT + lv], recs[out_sel],
                                   (const int32_t *)(ws + L.pool[lv]), rec_ints(width_of(lv)), out_sel ^ 1);
                    hio.is_helper = 1;
                    io.done = &ctr[CTR_DONE];
                    // entries are published by writing the task id: start from NO_TASK
                    if (cudaMemsetAsync(lists[out_sel], 0xff, sizeof(uint32_t) * (size_t)L.ntask, s) != cudaSuccess)
                        return LOGAN_ECUDA;
                }
                e = launch_width<FMT>(lv, latency_first, helpers, P, io, hio, sms, s, w0, w5, l1_g2);
            } else {
                io.max_count = latency_below;
                e = launch_width<FMT>(lv, true, false, P, io, io, sms, s, w0, w5);
                if (e == cudaSuccess) {
                    io.min_count = latency_below;
                    io.max_count = 0xffffffffu;
                    e = launch_width<FMT>(lv, false, false, P, io, io, sms, s, w0, w5);
                }
            }
        } else if (lv == BAND_LEVEL) {
          if constexpr (!no_band) {
            // stage 1: one warp per task, a 4096-slot ring; the bands that outgrow it
            // restart in stage 2 (four warps, 8192 slots), whose overflow goes on to level 8
            e = launch_band<FMT, BandSmall>(P, io, sms, s);
            if (e == cudaSuccess) {
                LevelIO io2 = io;
                io2.list = lists[out_sel];
                io2.count = &ctr[CTR_OUT + lv];
                io2.in_recs = nullptr;
                io2.rec_in = nullptr;
                io2.cursor = &ctr[CTR_BAND2_CURSOR];
                io2.out_list = lists[out_sel ^ 1];
                io2.out_count = &ctr[CTR_BAND2_OUT];
                e = launch_band<FMT, BandBig>(P, io2, sms, s);
                band2 = true;
            }
          }
        } else {
            if constexpr (fmt_base(FMT) == FMT_U8S)
                k_wide<FMT, SUBST_THREADS, true><<<WIDE_CTAS, SUBST_THREADS, 0, s>>>(P, io, wide, L.wide_stride);
            else
                k_wide<FMT><<<WIDE_CTAS, WIDE_THREADS, 0, s>>>(P, io, wide, L.wide_stride);
            e = cudaGetLastError();
        }
        if (e != cudaSuccess) return LOGAN_ECUDA;
        if (!mark(1 + lv, 1)) return LOGAN_ECUDA;
        in_list = band2 ? lists[out_sel ^ 1] : lists[out_sel];
        in_recs = (lv < NWIDTH) ? recs[out_sel] : nullptr;
        rec_in = (lv < NWIDTH) ? (const int32_t *)(ws + L.pool[lv]) : nullptr;
        rec_in_stride = (lv < NWIDTH) ? rec_ints(width_of(lv)) : 0;
        in_count = band2 ? &ctr[CTR_BAND2_OUT] : &ctr[CTR_OUT + lv];
        out_sel ^= 1;
        band2 = false;
    }
    int grid3 = (int)((P.n_pairs + per_block - 1) / per_block);
    if (grid3 > sms * 8) grid3 = sms * 8;
    if (grid3 < 1) grid3 = 1;
    if (!mark(LOGAN_N_STAGES - 1, 0)) return LOGAN_ECUDA;
    k_combine<FMT><<<grid3, SETUP_THREADS, 0, s>>>(P, tres, out, cells);
    if (cudaGetLastError() != cudaSuccess) return LOGAN_ECUDA;
    if (!mark(LOGAN_N_STAGES - 1, 1)) return LOGAN_ECUDA;
    return LOGAN_OK;
}

// explicit instantiations live in logan_fmt*.cu (one format per translation unit)
#define LOGAN_RUN_BATCH_SIG(F)                                                                   \
    int run_batch<F>(const Params &P, const logan_options_t *opt, bool wide_only, logan_result_t *out, \
                     uint64_t *cells, logan_stats_t *stats, uint8_t *ws, const Layout &L, cudaStream_t s)

}  // namespace logan

