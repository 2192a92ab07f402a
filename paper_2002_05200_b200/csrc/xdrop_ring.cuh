// xdrop_ring.cuh — the wide-band level: one warp per task, the two live
// antidiagonal arrays in a shared-memory RING indexed by diagonal slot.
//
// Same method and cell rule as the register windows (eq. P:85, drop rule P:89,
// best after the complete antidiagonal P:178, band trimming and termination
// P:186, c-amb-6/7), same threshold-relative values u = S - T_d and the same
// diagonal-slot coordinates (slot s on antidiagonal d is i = s + ceil(d/2),
// j = floor(d/2) - s; see xdrop_window.cuh). What changes is where the band
// lives, for bands too wide for registers (large X; the
// paper's X = 500 ... 5000 sweep):
//  * Each warp owns a ring of RING_SLOTS slots per parity in shared memory,
//    int16 per slot (live u <= X + match < 2^15 for X <= RING_XMAX; every dead
//    value is stored as -32768, which a step's rebase can never lift to >= 0,
//    and the cell's unsigned clamp re-kills it exactly). Slot s lives at ring
//    index s mod RING_SLOTS, so the band never has to be re-centred.
//  * Per antidiagonal the warp visits only the slots that can be live (the
//    predecessors' live extremes widened by one, clipped to the matrix) plus
//    the slots that were written two antidiagonals ago and are now outside
//    (they are cleared to dead, so everything outside the visited range of an
//    antidiagonal is dead: the invariant that makes reads outside it exact).
//    Lane l takes 8 consecutive slots of each 256-slot chunk: one 16-byte LDS
//    per array, the 8 cells in registers, one 16-byte STS back.
//  * The work per antidiagonal follows the band's width, with no window slack
//    and no barrier (one warp, __syncwarp between antidiagonals).
//  * A band wider than the ring (minus a margin) is handed to the CTA level
//    (restart); so is every task when X > RING_XMAX.
#pragma once

#include "xdrop_common.cuh"
#include "xdrop_window.cuh"

namespace logan {

constexpr int RING_SLOTS = 8192;                 // per parity, per warp
constexpr int RING_WARPS = 7;                    // warps (tasks) per block: 7 x 32 KB of smem
constexpr int RING_XMAX = 30000;                 // live u <= X + 127 must fit int16
constexpr int RING_MARGIN = 64;                  // slots kept free between the band's ends
constexpr uint32_t DEAD16X2 = 0x80008000u;       // two dead int16 slots
constexpr size_t RING_SMEM = (size_t)RING_WARPS * 2 * RING_SLOTS * sizeof(int16_t);

// 8 consecutive pool codes from position plo upwards (field q = position plo+q):
// 2-bit pool -> 8 2-bit fields in the low 16 bits; u8 pool -> 8 bytes.
template <int FMT> struct RingCodes;

template <> struct RingCodes<LOGAN_SEQ_2BIT> {
    uint32_t x;
    __device__ __forceinline__ void load(const Params &P, int64_t plo) {
        const int64_t w = plo >> 4;
        if (w >= 0 && w + 1 <= P.pool_words + 2) {  // the ABI's 16 readable bytes past the pool
            const uint32_t lo = __ldg(P.pool + w), hi = __ldg(P.pool + w + 1);
            x = __funnelshift_r(lo, hi, 2u * (uint32_t)(plo & 15)) & 0xffffu;
        } else {  // positions before the pool start: only out-of-range (masked) fields
            x = 0;
#pragma unroll 1
            for (int q = 0; q < 8; ++q) {
                const int64_t p = plo + q;
                if (p >= 0 && p < P.pool_len) x |= pool_base<LOGAN_SEQ_2BIT>(P, p) << (2 * q);
            }
        }
    }
    __device__ __forceinline__ void reverse() {  // field q <-> field 7-q
        uint32_t y = __brev(x) >> 16;
        x = ((y >> 1) & 0x5555u) | ((y & 0x5555u) << 1);
    }
    __device__ __forceinline__ static bool mis(const RingCodes &a, const RingCodes &b, int r) {
        return ((a.x ^ b.x) & (3u << (2 * r))) != 0;
    }
};

template <> struct RingCodes<LOGAN_SEQ_U8> {
    uint32_t lo, hi;
    __device__ __forceinline__ void load(const Params &P, int64_t plo) {
        const int64_t w = plo >> 2;
        if (w >= 0 && w + 2 <= P.pool_words + 2) {
            const uint32_t a = __ldg(P.pool + w), b = __ldg(P.pool + w + 1), c = __ldg(P.pool + w + 2);
            const uint32_t sh = 8u * (uint32_t)(plo & 3);
            lo = __funnelshift_r(a, b, sh);
            hi = __funnelshift_r(b, c, sh);
        } else {
            lo = hi = 0;
#pragma unroll 1
            for (int q = 0; q < 8; ++q) {
                const int64_t p = plo + q;
                if (p >= 0 && p < P.pool_len) {
                    const uint32_t v = pool_base<LOGAN_SEQ_U8>(P, p);
                    if (q < 4) lo |= v << (8 * q); else hi |= v << (8 * (q - 4));
                }
            }
        }
    }
    __device__ __forceinline__ void reverse() {
        const uint32_t t = lo;
        lo = __byte_perm(hi, 0, 0x0123);
        hi = __byte_perm(t, 0, 0x0123);
    }
    __device__ __forceinline__ static bool mis(const RingCodes &a, const RingCodes &b, int r) {
        return r < 4 ? ((a.lo ^ b.lo) & (0xffu << (8 * r))) != 0 : ((a.hi ^ b.hi) & (0xffu << (8 * (r - 4)))) != 0;
    }
};

// int16x2 <-> int32 (sign-extending; saturating on the way back)
__device__ __forceinline__ int32_t lo16(uint32_t w) { return (int32_t)(int16_t)(w & 0xffffu); }
__device__ __forceinline__ int32_t hi16(uint32_t w) { return (int32_t)w >> 16; }
__device__ __forceinline__ uint32_t pack16(int32_t lo, int32_t hi) {
    uint32_t r;  // d = sat16(hi) << 16 | sat16(lo)
    asm("cvt.pack.sat.s16.s32 %0, %1, %2;" : "=r"(r) : "r"(hi), "r"(lo));
    return r;
}

// Uniform (per-warp) state of one task.
struct RingTask {
    uint32_t task;
    SeqRef a, b;
    int32_t m, n, d;
    int32_t best, arg_i, arg_j;
    int32_t Tn, Tq[2];        // as in WinState: Tq[p] = T of the last antidiagonal of parity p
    int32_t sF[2], sL[2];     // live slot extremes of the last antidiagonal of each parity
    int32_t Dlo[2], Dhi[2];   // slots possibly non-dead in each parity's array
    uint64_t cells, cells_entry;
};

template <int FMT>
struct RingWarp {
    uint16_t *ring;  // this warp's 2 x RING_SLOTS int16 (parity p at ring + p*RING_SLOTS)
    int lane;
    RingTask t;

    __device__ __forceinline__ void clear() {
        uint4 *r4 = (uint4 *)ring;
        const uint4 z = make_uint4(DEAD16X2, DEAD16X2, DEAD16X2, DEAD16X2);
#pragma unroll 4
        for (int q = lane; q < 2 * RING_SLOTS / 8; q += 32) r4[q] = z;
        __syncwarp();
    }

    __device__ __forceinline__ void begin(const Params &P, uint32_t task) {
        const TaskDesc td = task_desc(P, task);
        t.task = task;
        t.a = td.a;
        t.b = td.b;
        t.m = td.a.len;
        t.n = td.b.len;
    }

    // fresh start at antidiagonal 0: the origin S(0,0) = 0, u = 0 - T_0 = X
    __device__ __forceinline__ void init(const Params &P, uint32_t task) {
        begin(P, task);
        t.d = 0;
        t.best = 0;
        t.arg_i = t.arg_j = 0;
        t.Tq[0] = t.Tq[1] = t.Tn = -P.xdrop;
        t.sF[0] = t.sL[0] = 0;
        t.sF[1] = EMPTY_F;
        t.sL[1] = EMPTY_L;
        t.Dlo[0] = t.Dhi[0] = 0;
        t.Dlo[1] = EMPTY_F;
        t.Dhi[1] = EMPTY_L;
        t.cells = t.cells_entry = 0;
        clear();
        if (lane == 0) ring[0] = (uint16_t)(int16_t)P.xdrop;
        __syncwarp();
    }

    // continue a task handed over by a register window (record layout: xdrop_window.cuh)
    __device__ __forceinline__ void resume(const Params &P, const int32_t *rec) {
        begin(P, (uint32_t)rec[0]);
        t.d = rec[1];
        const int32_t S0src = rec[2];
        t.best = rec[3]; t.arg_i = rec[4]; t.arg_j = rec[5];
        const bool odd = t.d & 1;
        t.Tn = rec[6];
        t.Tq[0] = odd ? rec[8] : rec[7];
        t.Tq[1] = odd ? rec[7] : rec[8];
        t.sF[0] = odd ? rec[11] : rec[9];
        t.sF[1] = odd ? rec[9] : rec[11];
        t.sL[0] = odd ? rec[12] : rec[10];
        t.sL[1] = odd ? rec[10] : rec[12];
        const int32_t Wsrc = rec[15];
        t.cells = (uint64_t)(uint32_t)rec[16] | ((uint64_t)(uint32_t)rec[17] << 32);
        t.cells_entry = t.cells;
        clear();
        for (int q = lane; q < Wsrc; q += 32) {
            const int32_t ri = (S0src + q) & (RING_SLOTS - 1);
            ring[ri] = (uint16_t)(int16_t)max(rec[REC_HDR + q], -32768);
            ring[RING_SLOTS + ri] = (uint16_t)(int16_t)max(rec[REC_HDR + Wsrc + q], -32768);
        }
        t.Dlo[0] = t.Dlo[1] = S0src;
        t.Dhi[0] = t.Dhi[1] = S0src + Wsrc - 1;
        __syncwarp();
    }

    // One antidiagonal d = t.d + 1 of parity PAR. Returns 0 = continue,
    // 1 = finished, 2 = band too wide for the ring.
    template <int PAR>
    __device__ __forceinline__ int step(const Params &P) {
        const int32_t d = t.d + 1;
        const int32_t ch = PAR ? (d + 1) >> 1 : d >> 1, fh = PAR ? (d - 1) >> 1 : d >> 1;
        const int32_t F1 = t.sF[1 - PAR], L1 = t.sL[1 - PAR], F2 = t.sF[PAR], L2 = t.sL[PAR];

        // (1) band cells of d (same count as the register windows, c-amb-14)
        {
            const int32_t c1 = PAR ? (d - 1) >> 1 : d >> 1;
            const int32_t c2 = PAR ? (d - 1) >> 1 : (d - 2) >> 1;
            const int32_t lo = max(min(F1 + c1, F2 + c2 + 1), max(1, d - t.n));
            const int32_t hi = min(max(L1 + c1, L2 + c2) + 1, min(t.m, d - 1));
            t.cells += (uint32_t)max(hi - lo + 1, 0);
        }

        // (2) slots that can be live: a live predecessor at d-1 (even d reads
        //     slots s-1 and s, odd d reads s and s+1) or d-2 (slot s), inside
        //     the matrix (0 <= i <= m, 0 <= j <= n)
        int32_t vlo = PAR ? min(F1 - 1, F2) : min(F1, F2);
        int32_t vhi = PAR ? max(L1, L2) : max(L1 + 1, L2);
        vlo = max(vlo, max(-ch, fh - t.n));
        vhi = min(vhi, min(t.m - ch, fh));
        // slots to write: the visited ones, and last time's ones (cleared)
        int32_t hlo = t.Dlo[PAR], hhi = t.Dhi[PAR];
        if (vlo <= vhi) { hlo = min(hlo, vlo); hhi = max(hhi, vhi); }

        // (3) rebased constants (see xdrop_window.cuh step (3))
        const int32_t Tc = t.Tn;
        const int32_t gp = P.gap - (Tc - t.Tq[1 - PAR]);
        const int32_t sma = P.match - (Tc - t.Tq[PAR]);
        const int32_t smi = P.mismatch - (Tc - t.Tq[PAR]);
        const int32_t fg = DEAD - gp;

        uint16_t *cur = ring + PAR * RING_SLOTS;        // d-2 in, d out (in place)
        const uint16_t *oth = ring + (1 - PAR) * RING_SLOTS;  // d-1
        const int32_t adir = t.a.dir, bdir = t.b.dir;
        const int64_t abase = t.a.base, bbase = t.b.base;

        int32_t run_u = -1, run_s = 0;          // this lane's best u and its (first) slot
        int32_t lf = INT32_MAX, ll = INT32_MIN; // this lane's live slot extremes
        if (hlo <= hhi) {
#pragma unroll 1
            for (int32_t c0 = hlo & ~7; c0 <= hhi; c0 += 256) {
                const int32_t s0 = c0 + 8 * lane;
                if (s0 > hhi) continue;
                const int32_t ri = s0 & (RING_SLOTS - 1);
                const int32_t rlo = vlo - s0, rhi = vhi - s0;  // visited fields of this lane: [rlo, rhi]
                uint4 out = make_uint4(DEAD16X2, DEAD16X2, DEAD16X2, DEAD16X2);
                if (rlo <= 7 && rhi >= 0) {
                    const uint4 dw = *(const uint4 *)(cur + ri);   // d-2 (diag)
                    const uint4 pw = *(const uint4 *)(oth + ri);   // d-1
                    const int32_t nb = (int32_t)(int16_t)oth[(PAR ? s0 + 8 : s0 - 1) & (RING_SLOTS - 1)];
                    const int32_t dg[8] = {lo16(dw.x), hi16(dw.x), lo16(dw.y), hi16(dw.y),
                                           lo16(dw.z), hi16(dw.z), lo16(dw.w), hi16(dw.w)};
                    const int32_t pv[8] = {lo16(pw.x), hi16(pw.x), lo16(pw.y), hi16(pw.y),
                                           lo16(pw.z), hi16(pw.z), lo16(pw.w), hi16(pw.w)};
                    // bases: slot s0+r holds a_{s0+r+ch} and b_{fh-s0-r}
                    RingCodes<FMT> ca, cb;
                    const int32_t ia = s0 + ch, jb = fh - s0;
                    ca.load(P, adir > 0 ? abase + ia - 1 : abase - ia - 6);
                    cb.load(P, bdir > 0 ? bbase + jb - 8 : bbase - jb + 1);
                    if (adir < 0) ca.reverse();
                    if (bdir > 0) cb.reverse();
                    int32_t u[8];
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        const int32_t p2 = PAR ? (r < 7 ? pv[r + 1] : nb) : (r > 0 ? pv[r - 1] : nb);
                        u[r] = Window<1, 1, FMT>::cell(pv[r], p2, dg[r], RingCodes<FMT>::mis(ca, cb, r), gp, fg,
                                                        sma, smi, P.one);
                    }
                    if (rlo > 0 || rhi < 7) {  // a band edge (or the matrix edge) cuts this lane
#pragma unroll
                        for (int r = 0; r < 8; ++r) u[r] = (r >= rlo && r <= rhi) ? u[r] : DEAD;
                    }
                    // argmax key u*9 + (7 - r): the max, then the smallest slot
                    int32_t kmax = INT32_MIN;
                    uint32_t dead = 0;
#pragma unroll
                    for (int r = 7; r >= 0; --r) {
                        kmax = max(kmax, u[r] * 9 + (7 - r));
                        dead = __funnelshift_l((uint32_t)u[r], dead, 1);  // bit r = sign of u[r]
                    }
                    const uint32_t live = ~dead & 0xffu;
                    if (live) {
                        lf = min(lf, s0 + __ffs(live) - 1);
                        ll = s0 + 31 - __clz(live);
                        const int32_t ku = kmax / 9;
                        if (ku > run_u) {  // strictly better than an earlier (lower) slot
                            run_u = ku;
                            run_s = s0 + 7 - (kmax - 9 * ku);
                        }
                    }
                    out = make_uint4(pack16(u[0], u[1]), pack16(u[2], u[3]), pack16(u[4], u[5]),
                                     pack16(u[6], u[7]));
                }
                *(uint4 *)(cur + ri) = out;
            }
        }
        __syncwarp();

        // (4) antidiagonal reductions: max u, its smallest slot, live extremes
        const int32_t M = __reduce_max_sync(0xffffffffu, run_u);
        const int32_t F = __reduce_min_sync(0xffffffffu, lf);
        const int32_t L = __reduce_max_sync(0xffffffffu, ll);
        if (M >= 0) {  // best after the complete antidiagonal, strict increase
            const int32_t V = M + Tc;
            if (V > t.best) {
                const int32_t slot = __reduce_min_sync(0xffffffffu, run_u == M ? run_s : INT32_MAX);
                t.best = V;
                t.arg_i = slot + ch;
                t.arg_j = d - t.arg_i;
            }
        }
        t.Tq[PAR] = Tc;
        t.Tn = t.best - P.xdrop;
        t.d = d;
        const bool h = F != INT32_MAX;
        t.sF[PAR] = h ? F : EMPTY_F;
        t.sL[PAR] = h ? L : EMPTY_L;
        t.Dlo[PAR] = vlo <= vhi ? vlo : EMPTY_F;
        t.Dhi[PAR] = vlo <= vhi ? vhi : EMPTY_L;

        // (5) termination: d and d-1 both empty (c-amb-7)
        if (t.sF[0] == EMPTY_F && t.sF[1] == EMPTY_F) return 1;
        // (6) the next antidiagonal touches at most the span of both arrays'
        //     written slots widened by 9 on each side: it must fit the ring
        const int32_t lo = min(t.Dlo[0], t.Dlo[1]), hi = max(t.Dhi[0], t.Dhi[1]);
        if (hi - lo + 1 > RING_SLOTS - RING_MARGIN) return 2;
        return 0;
    }
};

// Persistent kernel: each warp pulls tasks (or hand-over records) from the
// level's list and sweeps them to the end; overflow goes to the next level.
template <int FMT>
__global__ void __launch_bounds__(RING_WARPS * 32, 1) k_ring(const Params P, const LevelIO io) {
    extern __shared__ uint4 ring_smem[];
    RingWarp<FMT> w;
    w.lane = threadIdx.x & 31;
    w.ring = (uint16_t *)ring_smem + (size_t)(threadIdx.x >> 5) * 2 * RING_SLOTS;
    const uint32_t count = *io.count;
    for (;;) {
        uint32_t pos = 0;
        if (w.lane == 0) pos = atomicAdd(io.cursor, 1u);
        pos = __shfl_sync(0xffffffffu, pos, 0);
        if (pos >= count) return;
        const uint32_t task = io.list[pos];
        int rc = 2;
        if (P.xdrop <= RING_XMAX) {
            const uint32_t rec = io.in_recs ? io.in_recs[pos] : NO_REC;
            if (rec != NO_REC) w.resume(P, io.rec_in + (size_t)rec * io.rec_in_stride);
            else w.init(P, task);
            if (io.stats && w.lane == 0)
                atomicAdd((unsigned long long *)&io.stats->tasks_started[io.level], 1ull);
            do {
                rc = (w.t.d & 1) ? w.template step<0>(P) : w.template step<1>(P);
            } while (rc == 0);
        }
        if (w.lane == 0) {
            if (rc == 1) {
                TaskRes tr;
                tr.best = w.t.best;
                tr.i = w.t.arg_i;
                tr.j = w.t.arg_j;
                tr.flags = 0;
                tr.cells = w.t.cells;
                io.tres[task] = tr;
                if (io.stats) {
                    atomicAdd((unsigned long long *)&io.stats->tasks_finished[io.level], 1ull);
                    atomicAdd((unsigned long long *)&io.stats->cells_per_level[io.level],
                              (unsigned long long)(w.t.cells - w.t.cells_entry));
                    atomicAdd((unsigned long long *)&io.stats->cells_total, (unsigned long long)w.t.cells);
                }
            } else {  // the CTA level restarts it from antidiagonal 0
                const uint32_t o = atomicAdd(io.out_count, 1u);
                io.out_list[o] = task;
            }
        }
    }
}

}  // namespace logan
