// xdrop_window.cuh — the hot path: X-drop antidiagonal sweep in a register
// window (sm_100a, integer SIMT, no tensor cores).
//
// Method (§III-A, Alg. 1, Alg. 2):
// each cell S(i,j) = max(diag + s(a_i,b_j), up + gap, left + gap) over live
// predecessors (eq. P:85); a cell with S < best - X is dead for good;
// best is updated once the antidiagonal is complete; the band is
// trimmed to the cells that can still have a live predecessor and the
// extension stops when two consecutive antidiagonals are empty (P:186,
// c-amb-6/7).
//
// B200 design, not the paper's V100 one:
//  * Cells are addressed by DIAGONAL SLOT s = floor((i - j) / 2) instead of by
//    column: on antidiagonal d, slot s is the cell i = s + ceil(d/2),
//    j = floor(d/2) - s. The X-drop band follows the alignment's diagonal, so
//    in slot space it stays put (it drifts only with net indels) and a fixed
//    register window of W = G*R slots holds it: G lanes per task, R slots per
//    lane, two register arrays E[] (even antidiagonal) and O[] (odd one).
//    Predecessors of slot s: even d: up = O[s], left = O[s-1], diag = E[s];
//    odd d: up = E[s+1], left = E[s], diag = O[s]. Each step overwrites the
//    array of its parity in place; only the lane-boundary value crosses lanes
//    (one SHFL per step).
//  * Scores are stored RELATIVE to a kill threshold T_e = best_{e-1} - X, and
//    the kill is applied ONE ANTIDIAGONAL LATE ("kill on read"): step e first
//    kills antidiagonal e-1 with T_{e-1} (one VIADDMNMX.U32 per slot, which also
//    rebases it: u = min_u32(u' - (T_{e-1} - T_{e-2}), DEAD)), then computes the
//    RAW cells of e from the killed e-1 and e-2 (relative to T_{e-1}):
//        u' = max(max(up, left, DEAD - gap) + gap, diag + s - (T_{e-1} - T_{e-2}))
//    (VIMNMX3, an FMA-pipe IMAD for diag + s', VIADDMNMX). best_e is the max
//    over raw e (a raw value above best_{e-1} is >= T_e, i.e. live), so the
//    reduction of e's maximum only has to finish by step e + 2: it overlaps
//    step e + 1 instead of sitting on the per-antidiagonal critical path
//    (for a warp per task: CREDUX ~23 cycles, measured in tools/lat_probe.cu).
//    Every negative value after the kill is dead, and DEAD - 3*127 <= dead
//    values <= DEAD (the floor keeps raw values >= DEAD): exact and absorbing.
//  * Bases sit in registers, 4-bit fields (2-bit pool) or 16-bit fields (u8
//    pool), one per slot; positions past an extension's end hold sentinels
//    that match nothing, so cells outside the matrix (i > m or j > n) can only
//    hold values below an earlier best and are excluded from the band
//    bookkeeping by a per-lane validity mask -- no per-cell masking.
//  * Per antidiagonal the max and its slot come from one packed key
//    (u' * 1027 + 1023 - slot, an IMAD) reduced with VIMNMX3 inside the lane and
//    CREDUX / SHFL butterflies across the G lanes; it is decoded only when it
//    raises best. The live extremes come from a funnel-shifted sign mask + FLO.
//    Ties go to the smallest slot = smallest i (c-amb-9).
//  * The window re-centres by one slot when the band touches an edge; if the
//    band is wider than W - 2 slots the task is handed to the next level in the
//    canonical (un-pipelined) state after an even antidiagonal.
#pragma once

#include <type_traits>

#include "xdrop_common.cuh"

namespace logan {

constexpr int32_t DEAD = -(1 << 20);
constexpr uint32_t DEADU = 0xFFF00000u;  // (uint32_t)DEAD
// Argmax key of a cell: u * KEYMUL + (1023 - slot). KEYMUL > 1023 keeps the
// order (value, then smallest slot); it is not a power of two so the key is
// one IMAD on the FMA pipe (the ALU pipe is the kernel's bottleneck).
// |DEAD - 1024| * KEYMUL < 2^31 and (X + 3*127) * KEYMUL < 2^31 for X <= 2^19.
constexpr int32_t KEYMUL = 1027;
constexpr int32_t KNONE = INT32_MIN;  // "no pending maximum" (below every raise threshold)

// Minimum resident blocks per SM requested for the one-lane-per-task kernels
// (caps registers; tuned by measurement).
#ifndef LOGAN_L0_MINB
#define LOGAN_L0_MINB 1
#endif
// the same for the packed first window (Window16; see LOGAN_PK_HSHAPE) with 28 or 32
// slots; 24 slots and fewer take 4 blocks (128 registers, no spill): C3 X = 10 +3.5%,
// while 4 blocks cost 32 slots 5% (profiles/r02/ab_minb4.txt)
#ifndef LOGAN_PK_MINB
#define LOGAN_PK_MINB 1
#endif

#ifndef LOGAN_NCHAIN
#define LOGAN_NCHAIN 4
#endif

template <int FMT> struct RegFmt;
template <> struct RegFmt<LOGAN_SEQ_2BIT> {
    static constexpr int CB = 4;                 // bits per register field
    static constexpr uint32_t SA = 4u, SB = 8u;  // sentinels past the ends of A / B
    // field of a base (or sentinel) entering the A / B registers
    __device__ __forceinline__ static uint32_t fa(uint32_t x) { return x; }
    __device__ __forceinline__ static uint32_t fb(uint32_t x) { return x; }
};
template <> struct RegFmt<LOGAN_SEQ_U8> {
    static constexpr int CB = 16;
    static constexpr uint32_t SA = 0x100u, SB = 0x200u;
    __device__ __forceinline__ static uint32_t fa(uint32_t x) { return x; }
    __device__ __forceinline__ static uint32_t fb(uint32_t x) { return x; }
};
// Substitution-matrix scoring: an A field holds code << 6, a B field the code
// (both mod 32), so A + B of two packed words is two table indices at once;
// the sentinels are row / column 32 of the table (load_subst_tab).
template <> struct RegFmt<FMT_U8S> {
    static constexpr int CB = 16;
    static constexpr uint32_t SA = 0x100u, SB = 0x100u;  // raw sentinels (> any byte); fa / fb map them to 32
    __device__ __forceinline__ static uint32_t fa(uint32_t x) { return x < 256u ? (x & 31u) << 6 : 32u << 6; }
    __device__ __forceinline__ static uint32_t fb(uint32_t x) { return x < 256u ? (x & 31u) : 32u; }
};
template <> struct RegFmt<LOGAN_SEQ_2BIT | FMT_Z> : RegFmt<LOGAN_SEQ_2BIT> {};
template <> struct RegFmt<LOGAN_SEQ_U8 | FMT_Z> : RegFmt<LOGAN_SEQ_U8> {};
template <> struct RegFmt<FMT_U8S | FMT_Z> : RegFmt<FMT_U8S> {};

// Group-uniform state of one task (replicated in each lane of the group), in
// the PIPELINED form of the sweep (header, "kill one antidiagonal late"). At
// the start of step e (computing antidiagonal e; d = e - 1):
//   - array of parity (e-1)&1: RAW values of e-1, relative to T_{e-2};
//   - array of parity e&1:     KILLED values of e-2, relative to T_{e-2};
//   - best / arg: folded through antidiagonal e-3 (best_{e-3});
//   - Tq[(e-2)&1] = T_{e-2}; Tq[(e-1)&1] = T_{e-3};
//   - K[(e-2)&1], K[(e-1)&1]: the pending maxima (keys) of raw e-2 and e-1
//     (KNONE once folded), relative to T_{e-3} and T_{e-2};
//   - sF / sL[(e-2)&1]: live slot extremes of e-2; [(e-1)&1] of e-3 (stale).
template <int FMT>
struct WinState {
    // sa feeds the top slot (read by lane G-1; sa.idx = S0 + W + ceil(d/2)),
    // sb feeds the bottom slot (read by lane 0; sb.idx = floor(d/2) - S0 + 1)
    Stream<FMT> sa, sb;
    uint32_t task;
    int32_t m, n;
    int32_t d;             // last antidiagonal whose raw values are computed
    int32_t S0;            // slot of the window's first register
    int32_t best, arg_i, arg_j;
    int32_t Tq[2];
    int32_t K[2];
    int32_t KZ[2];         // Z-drop builds: pending in-matrix maxima (keys)
    uint32_t dc[2];        // Z-drop builds: band cells added for the last antidiagonal of each parity
    // an antidiagonal without a (valid) live cell has sF = EMPTY_F, sL =
    // EMPTY_L, which makes every min / max below ignore it without a branch
    int32_t sF[2], sL[2];
    uint64_t cells;
    uint64_t cells_entry;  // cells already counted when the task entered this level
    uint32_t shifts;
};

// Hand-over record between levels: REC_HDR ints of scalars, then E[W], O[W].
// The record holds the CANONICAL state after antidiagonal d (both d and d-1
// killed; best = best_d), the format every level reads.
constexpr int REC_HDR = 32;
__host__ __device__ constexpr int rec_ints(int W) { return REC_HDR + 2 * W; }
constexpr uint32_t NO_REC = 0xffffffffu;
constexpr int32_t EMPTY_F = 1 << 29, EMPTY_L = -(1 << 29);

// Reductions over the G lanes of a group: one CREDUX for a full warp,
// SHFL butterflies for sub-warp groups.
template <int G>
__device__ __forceinline__ int32_t grp_max(int32_t v, unsigned gmask) {
    if (G == 32) return __reduce_max_sync(0xffffffffu, v);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(gmask, v, o, G));
    return v;
}
template <int G>
__device__ __forceinline__ int32_t grp_min(int32_t v, unsigned gmask) {
    if (G == 32) return __reduce_min_sync(0xffffffffu, v);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(gmask, v, o, G));
    return v;
}

// min_u32(a + b, c): VIADDMNMX.U32 (the late kill, one DPX op)
__device__ __forceinline__ uint32_t addmin_u32(uint32_t a, uint32_t b, uint32_t c) { return __viaddmin_u32(a, b, c); }

template <int G, int R, int FMT>
struct Window {
    using RF = RegFmt<FMT>;
    static constexpr int CB = RF::CB;
    static constexpr int FPW = 32 / CB;             // fields per word
    static constexpr int NW = (R + FPW - 1) / FPW;  // words per lane per sequence
    static constexpr int RL = R - (NW - 1) * FPW;   // fields in the last word
    static constexpr int W = G * R;
    static constexpr int GG = G;
    static constexpr uint32_t FM = (1u << CB) - 1u;
    static constexpr bool ZON = fmt_z(FMT);
    static_assert(R >= 1 && R <= 32 && W <= 1024 && (G & (G - 1)) == 0, "window shape");

    int32_t E[R], O[R];
    uint32_t Aw[NW], Bw[NW];
    WinState<FMT> st;
    int gl;            // lane within group
    unsigned gmask;

    // RAW cell (eq. P:85) on values relative to T_{e-1}: up / left are killed
    // values of e-1 (relative to T_{e-1}), diag a killed value of e-2; the
    // diagonal term carries the rebase T_{e-2} - T_{e-1} inside sma / smi.
    //   u' = max(max(up, left, fg) + gap, diag + s')   (fg = DEAD - gap: a floor)
    // The kill is applied one antidiagonal later (kill_u).
    // Substitution-matrix cell: s = the table entry, sr = the diagonal rebase.
    __device__ __forceinline__ static int32_t cell_s(int32_t up, int32_t left, int32_t diag, int32_t s,
                                                     int32_t gp, int32_t fg, int32_t sr) {
        const int32_t t0 = __vimax3_s32(up, left, fg);
        return __viaddmax_s32(t0, gp, diag + s + sr);
    }
    const int8_t *tab;  // FMT_U8S: the substitution table in shared memory

    // The kernel is bound by the ALU pipe (VIMNMX3, VIADDMNMX and the kill live
    // there), so diag + s' is computed on the FMA pipe: an IMAD by an opaque
    // run-time 1 for the match case, overwritten by a predicated IMAD for a
    // mismatch -- no SEL, no IADD3.
    __device__ __forceinline__ static int32_t cell(int32_t up, int32_t left, int32_t diag, bool mis,
                                                   int32_t gp, int32_t fg, int32_t sma, int32_t smi,
                                                   int32_t one) {
        const int32_t t0 = __vimax3_s32(up, left, fg);
        int32_t dps;
        asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(dps) : "r"(diag), "r"(one), "r"(sma));
        asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q mad.lo.s32 %0, %2, %3, %4;\n\t}"
            : "+r"(dps) : "r"((uint32_t)mis), "r"(diag), "r"(one), "r"(smi));
        return __viaddmax_s32(t0, gp, dps);
    }
    // The late kill: a raw value of e relative to T_{e-1} becomes a killed value
    // relative to T_e (dl = T_e - T_{e-1} >= 0): u = u' - dl if u' - dl >= 0,
    // else a dead value in [DEAD - 3*127, DEAD] (every negative u' - dl >= DEAD
    // maps to exactly DEAD; the floor fg keeps raw values >= DEAD).
    __device__ __forceinline__ static int32_t kill_u(int32_t u, int32_t ndl) {
        return (int32_t)addmin_u32((uint32_t)u, (uint32_t)ndl, DEADU);
    }

    // per-thread shared-memory slice used only by the (rare) window shifts
    static constexpr int SB_STRIDE = 2 * R + 1;  // odd stride: conflict-free
    int32_t *sbase;
    __device__ __forceinline__ volatile int32_t *sbuf() const { return sbase; }
    __device__ __forceinline__ void spill(const int32_t (&e)[R], const int32_t (&o)[R]) const {
        volatile int32_t *b = sbase;
#pragma unroll
        for (int r = 0; r < R; ++r) { b[r] = e[r]; b[R + r] = o[r]; }
    }

    // ---- field helpers ------------------------------------------------------
    __device__ __forceinline__ uint32_t field(const uint32_t (&w)[NW], int r) const {
        return (w[r / FPW] >> (CB * (r % FPW))) & FM;
    }
    // the top field (slot R-1) of a lane's word array
    __device__ __forceinline__ static uint32_t top_field(const uint32_t (&w)[NW]) {
        return (w[NW - 1] >> (CB * (RL - 1))) & FM;
    }
    // fields r <- r+1, new value into the top field (bits above it stay zero)
    __device__ __forceinline__ static void shift_down(uint32_t (&w)[NW], uint32_t in) {
#pragma unroll
        for (int q = 0; q < NW - 1; ++q) w[q] = __funnelshift_r(w[q], w[q + 1], CB);
        if (RL == FPW) w[NW - 1] = __funnelshift_r(w[NW - 1], in, CB);
        else w[NW - 1] = (w[NW - 1] >> CB) | (in << (CB * (RL - 1)));
    }
    // fields r <- r-1, new value into field 0
    __device__ __forceinline__ static void shift_up(uint32_t (&w)[NW], uint32_t in) {
#pragma unroll
        for (int q = NW - 1; q > 0; --q) w[q] = __funnelshift_l(w[q - 1], w[q], CB);
        w[0] = (w[0] << CB) | in;
        if (RL < FPW) w[NW - 1] &= (1u << (CB * (RL < FPW ? RL : 0))) - 1u;
    }

    // ---- task start -----------------------------------------------------------
    // Pipelined state before step e = 1: raw antidiagonal 0 (the origin,
    // relative to T_{-1} = -X: u' = X), killed antidiagonal -1 (all dead),
    // nothing pending.
    __device__ __forceinline__ void init(const Params &P, uint32_t task) {
        const TaskDesc td = task_desc(P, task);
        st.task = task;
        st.m = td.a.len;
        st.n = td.b.len;
        st.d = 0;
        st.S0 = -(W / 2);
        st.best = 0;  // best_{-2} := 0
        st.arg_i = st.arg_j = 0;
        st.Tq[0] = st.Tq[1] = -P.xdrop;  // T_{-1} = T_{-2} = 0 - X
        st.K[0] = st.K[1] = KNONE;
        st.KZ[0] = st.KZ[1] = KNONE;
        st.dc[0] = st.dc[1] = 0;
        st.sF[1] = EMPTY_F;  // antidiagonal -1: empty
        st.sL[1] = EMPTY_L;
        st.sF[0] = EMPTY_F;  // antidiagonal 0: set by step 1's kill
        st.sL[0] = EMPTY_L;
        st.cells = 0;
        st.shifts = 0;
        const int32_t s0 = st.S0 + gl * R;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            E[r] = (s0 + r == 0) ? P.xdrop : DEAD;
            O[r] = DEAD;
        }
        st.sa.s = td.a;
        st.sb.s = td.b;
        st.cells_entry = 0;
        load_bases(P);
    }

    // bases of the window at antidiagonal st.d: slot s holds a_{s + ceil(d/2)}
    // and b_{floor(d/2) - s}; positions the top / bottom streams (rolled loops:
    // runs once per task start or resume)
    __device__ __forceinline__ void load_bases(const Params &P) {
        const int32_t s0 = st.S0 + gl * R;
        const int32_t ch = ceil_half(st.d), fh = floor_half(st.d);
#pragma unroll
        for (int q = 0; q < NW; ++q) { Aw[q] = 0; Bw[q] = 0; }
        st.sa.seek(P, s0 + ch);
#pragma unroll 1
        for (int r = 0; r < R; ++r) shift_down(Aw, RF::fa(st.sa.next(P, RF::SA)));  // field r = a_{s0+r+ch}
        st.sb.seek(P, fh - (s0 + R - 1));
#pragma unroll 1
        for (int r = R - 1; r >= 0; --r) shift_up(Bw, RF::fb(st.sb.next(P, RF::SB)));  // field r = b_{fh-(s0+r)}
        if (gl == G - 1) st.sa.seek(P, st.S0 + W + ch);  // sa.idx = S0 + W + ceil(d/2)
        if (gl == 0) st.sb.seek(P, fh - st.S0 + 1);      // sb.idx = floor(d/2) - S0 + 1
    }

    // the argmax is decoded at each raise (nothing pending at the task's end)
    __device__ __forceinline__ void finalize() {}

    // ---- pending maxima -------------------------------------------------------
    // Fold the pending key k of raw antidiagonal a (relative to threshold T, with
    // the window base S0) into best: V = ku + T, a raise only on a strict
    // increase, argmax = that slot (c-amb-8/9).
    __device__ __forceinline__ void fold(int32_t k, int32_t T, int32_t a) {
        if (k >= (st.best - T + 1) * KEYMUL) {  // the decode runs only on antidiagonals that raise best
            const int32_t ku = k / KEYMUL;
            st.best = ku + T;
            st.arg_i = st.S0 + (1023 - (k - ku * KEYMUL)) + ceil_half(a);
            st.arg_j = a - st.arg_i;
        }
    }
    // Z-drop test (c-amb-19) of antidiagonal a with best = best_a already
    // folded: kz = the pending in-matrix key of raw a (relative to T), live iff
    // its value is >= Ta; stop if best - M_a > Z + |gap| * |(i_a - i*) - (j_a - j*)|.
    // Every live M_a is >= Ta = best_{a-1} - X, so a stop needs M_a < best - Z
    // (cheap pre-test first).
    __device__ __forceinline__ bool zstop(const Params &P, int32_t kz, int32_t T, int32_t Ta, int32_t a) const {
        if (kz < (Ta - T) * KEYMUL || kz >= (st.best - P.zdrop - T) * KEYMUL) return false;
        const int32_t kzu = kz / KEYMUL;
        const int32_t zi = st.S0 + (1023 - (kz - kzu * KEYMUL)) + ceil_half(a);
        const int32_t off = abs((zi - st.arg_i) - ((a - zi) - st.arg_j));
        return st.best - (kzu + T) > P.zdrop - P.gap * off;
    }

    // ---- exact hand-over between levels ---------------------------------------
    // Called at the check point of an odd step e (after the kill of e-1, with
    // e-1's pending raw maximum folded by the step): the canonical state after
    // antidiagonal d = e - 1 is written (values of d and d-1, both killed;
    // best = best_d), and the next, wider level continues it from d + 1: cells
    // outside the old window are dead (the band invariant), so the continuation
    // is exact. The value arrays are stored by parity (E, then O).
    __device__ __forceinline__ void save(const Params &P, int32_t *rec) const {
        const int32_t d = st.d;
        const int p = d & 1;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            rec[REC_HDR + gl * R + r] = E[r];
            rec[REC_HDR + W + gl * R + r] = O[r];
        }
        if (gl == 0) {
            rec[0] = (int32_t)st.task; rec[1] = d; rec[2] = st.S0; rec[3] = st.best;
            rec[4] = st.arg_i; rec[5] = st.arg_j;
            // (parity-indexed state through selects: a run-time index would put
            // the arrays in local memory)
            rec[6] = st.best - P.xdrop;                       // T_{d+1}
            rec[7] = p ? st.Tq[1] : st.Tq[0];                 // T_d
            rec[8] = p ? st.Tq[0] : st.Tq[1];                 // T_{d-1}
            rec[9] = p ? st.sF[1] : st.sF[0];                 // extremes of d
            rec[10] = p ? st.sL[1] : st.sL[0];
            rec[11] = p ? st.sF[0] : st.sF[1];                // extremes of d-1
            rec[12] = p ? st.sL[0] : st.sL[1];
            rec[13] = 0;
            rec[14] = (int32_t)st.shifts; rec[15] = W;
            rec[16] = (int32_t)(uint32_t)st.cells; rec[17] = (int32_t)(uint32_t)(st.cells >> 32);
        }
    }

    // Resume from the canonical record after antidiagonal d into the pipelined
    // state before step e = d + 1: killed d is re-expressed as raw relative to
    // T_{d-1} (u + T_d - T_{d-1}; the late kill at step e restores it exactly),
    // best := best_{d-1} = T_d + X, and a raise on d (best_d > best_{d-1}, at the
    // recorded argmax, which then lies on d) is re-issued as d's pending key.
    __device__ __forceinline__ void resume(const Params &P, const int32_t *rec) {
        st.task = (uint32_t)rec[0];
        const TaskDesc td = task_desc(P, st.task);
        st.m = td.a.len;
        st.n = td.b.len;
        st.sa.s = td.a;
        st.sb.s = td.b;
        const int32_t d = rec[1];
        st.d = d;
        const int32_t S0src = rec[2];
        const int32_t best_d = rec[3];
        st.arg_i = rec[4]; st.arg_j = rec[5];
        const int32_t Td = rec[7], Td1 = rec[8];
        const int p = d & 1;
        st.Tq[0] = st.Tq[1] = Td1;  // T_{e-2} = T_{d-1}; T_{e-3} only decodes K[1-p] = KNONE
        st.best = Td + P.xdrop;     // best_{d-1}
        st.sF[0] = p ? rec[11] : rec[9];
        st.sL[0] = p ? rec[12] : rec[10];
        st.sF[1] = p ? rec[9] : rec[11];
        st.sL[1] = p ? rec[10] : rec[12];
        st.shifts = (uint32_t)rec[14];
        const int32_t Wsrc = rec[15];
        st.cells = (uint64_t)(uint32_t)rec[16] | ((uint64_t)(uint32_t)rec[17] << 32);
        st.cells_entry = st.cells;
        st.KZ[0] = st.KZ[1] = KNONE;
        st.dc[0] = st.dc[1] = 0;
        // centre the wider window on the live band of d and d-1
        int32_t Fm = min(st.sF[0], st.sF[1]), Lm = max(st.sL[0], st.sL[1]);
        if (Fm > Lm) { Fm = S0src; Lm = S0src + Wsrc - 1; }
        st.S0 = ((Fm + Lm) >> 1) - W / 2;
        const int32_t kd = best_d > st.best
                               ? (best_d - Td1) * KEYMUL + (1023 - (st.arg_i - ceil_half(d) - st.S0)) : KNONE;
        st.K[0] = p ? KNONE : kd;
        st.K[1] = p ? kd : KNONE;
        const int32_t rb = Td - Td1;  // killed d (relative to T_d) as raw relative to T_{d-1}
        const int32_t s0 = st.S0 + gl * R;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int32_t q = s0 + r - S0src;
            const bool in = q >= 0 && q < Wsrc;
            const int32_t ve = in ? rec[REC_HDR + q] : DEAD;         // even array
            const int32_t vo = in ? rec[REC_HDR + Wsrc + q] : DEAD;  // odd array
            E[r] = p == 0 ? ve + rb : ve;
            O[r] = p == 1 ? vo + rb : vo;
        }
        load_bases(P);
    }

    // ---- one pipelined step: antidiagonal e = st.d + 1 of parity PAR ----------
    // (a) fold the pending raw maximum of e-2 -> best_{e-2}, T_{e-1};
    // (b) kill e-1 with T_{e-1} (its live extremes);
    // (c) odd e only: termination (e-1 and e-2 empty) and the window check;
    // (d) the band cells of e; (e) bases of e; (f) raw e; (g) its maximum,
    // left pending (reduced across the group while the next step runs).
    // Returns 0 = continue, 1 = finished, 2 = overflow (hand over).
    template <int PAR>
    __device__ __forceinline__ int step(const Params &P, bool force) {
        const int32_t e = st.d + 1;
        constexpr int Q = 1 - PAR;  // parity of e-1 (array E for odd e, O for even e)

        // (a) best_{e-2} from the raw maximum of e-2 (relative to T_{e-3} = Tq[Q])
        fold(st.K[PAR], st.Tq[Q], e - 2);
        st.K[PAR] = KNONE;
        const int32_t T1 = st.best - P.xdrop;  // T_{e-1}
        const int32_t T2 = st.Tq[PAR];         // T_{e-2}
        if (ZON && P.zdrop >= 0) {
            if (zstop(P, st.KZ[PAR], st.Tq[Q], T2, e - 2)) {
                st.cells -= st.dc[Q];  // the sweep ends after e-2: e-1's band was counted already
                return 1;
            }
            st.KZ[PAR] = KNONE;
        }
        const int32_t dl = T1 - T2;  // >= 0

        // (b) late kill of e-1 (dead iff S < best_{e-2} - X), sign masks
        constexpr int NCH = LOGAN_NCHAIN;  // independent dead-mask chains per lane
        constexpr int RQ = (R + NCH - 1) / NCH;
        uint32_t dq[NCH];
#pragma unroll
        for (int r = R - 1; r >= 0; --r) {
            int32_t u;
            if (PAR) { u = kill_u(E[r], -dl); E[r] = u; }
            else { u = kill_u(O[r], -dl); O[r] = u; }
            const int c = r / RQ;
            const bool top = (r == R - 1) || (r == (c + 1) * RQ - 1);
            dq[c] = top ? ((uint32_t)u >> 31) : __funnelshift_l((uint32_t)u, dq[c], 1);
        }
        uint32_t dead = 0;
#pragma unroll
        for (int c = 0; c < NCH; ++c)
            if (c * RQ < R) dead |= dq[c] << (c * RQ);
        {
            // validity of slots on e-1: i <= m <=> s <= m - ceil((e-1)/2),
            // j <= n <=> s >= floor((e-1)/2) - n (cells with i < 0 or j < 0 are
            // dead by construction)
            const int32_t chq = e >> 1, fhq = (e - 1) >> 1;  // ceil((e-1)/2), floor((e-1)/2)
            const int32_t vlo = fhq - st.n, vhi = st.m - chq;
            const int32_t base = st.S0 + gl * R;
            uint32_t vmask = (R == 32) ? 0xffffffffu : ((1u << R) - 1u);
            if (vlo > base || vhi < base + R - 1) {
                const int32_t rlo = max(vlo - base, 0), rhi = min(vhi - base, R - 1);
                vmask = (rlo <= rhi) ? ((0xffffffffu >> (31 - rhi)) & ~((1u << rlo) - 1u)) : 0u;
            }
            const uint32_t live = ~dead & vmask;
            if (G == 1) {  // one lane per task: extremes only read when live != 0
                const bool h = live != 0;
                st.sF[Q] = h ? base + __ffs(live) - 1 : EMPTY_F;
                st.sL[Q] = h ? base + 31 - __clz(live) : EMPTY_L;
            } else {
                int32_t lf = live ? gl * R + __ffs(live) - 1 : INT32_MAX;
                int32_t ll = live ? gl * R + 31 - __clz(live) : INT32_MIN;
                lf = grp_min<G>(lf, gmask);
                ll = grp_max<G>(ll, gmask);
                const bool h = lf != INT32_MAX;
                st.sF[Q] = h ? st.S0 + lf : EMPTY_F;
                st.sL[Q] = h ? st.S0 + ll : EMPTY_L;
            }
        }
        st.Tq[Q] = T1;

        // (c) after an even antidiagonal e-1 (odd e): termination -- antidiagonals
        // e-1 and e-2 both empty (c-amb-7); best_{e-2} is final (a raw
        // value of e-1 above best_{e-2} would have been live) -- and the window:
        // the band's right edge can grow (by one slot) only on even antidiagonals
        // and its left edge only on odd ones, so the margin-1 invariant checked
        // here keeps every cell outside the window dead through the next two.
        if (PAR == 1) {
            if (st.sF[0] == EMPTY_F && st.sF[1] == EMPTY_F) return 1;
            bool ho = force;  // force: test knob (options.handover)
            if (!ho) {
                // keep the live band of e-1 and e-2 inside [S0+1, S0+W-2]
                const int32_t Fm = min(st.sF[0], st.sF[1]), Lm = max(st.sL[0], st.sL[1]);
                const bool lowv = Fm < st.S0 + 1, highv = Lm > st.S0 + W - 2;
                if (lowv || highv) {
                    if (lowv && highv) ho = true;
                    else if (lowv) {
                        if (Lm > st.S0 + W - 3) ho = true;
                        else shift_left(P, e - 1);
                    } else {
                        if (Fm < st.S0 + 2) ho = true;
                        else shift_right(P, e - 1);
                    }
                }
            }
            if (ho) {  // hand over the canonical state after e-1 (save): fold e-1's maximum
                fold(st.K[Q], T2, e - 1);
                st.K[Q] = KNONE;
                if (ZON && P.zdrop >= 0 && zstop(P, st.KZ[Q], T2, T1, e - 1)) return 1;
                return 2;
            }
        }

        // (d) band cells of e from the live extremes of e-1, e-2 (c-amb-14:
        //     lo = max(1, e-n, min(F1, F2+1)), hi = min(m, e-1, max(L1, L2)+1)).
        //     Empty antidiagonals carry EMPTY_F / EMPTY_L and drop out of the
        //     min / max; e = 1 clips to an empty band by itself.
        {
            // column of slot 0 on e-1 (c1) and e-2 (c2 = c1 - 1 + PAR), so with
            // c = c1: odd e: lo = max(min(F1, F2 + 1) + c, 1, e-n), hi = min(max(L1, L2) + c + 1, m, e-1);
            // even e: lo = max(min(F1, F2) + c, 1, e-n), hi = min(max(L1, L2 - 1) + c + 1, m, e-1)
            const int32_t c = PAR ? (e - 1) >> 1 : e >> 1;
            const int32_t F1 = st.sF[Q], F2 = st.sF[PAR], L1 = st.sL[Q], L2 = st.sL[PAR];
            const int32_t fmin = PAR ? min(F1, F2 + 1) : min(F1, F2);
            const int32_t lmax = PAR ? max(L1, L2) : max(L1, L2 - 1);
            const int32_t lo = __vimax3_s32(fmin + c, 1, e - st.n);
            const int32_t hi = __vimin3_s32(lmax + c + 1, st.m, e - 1);
            const uint32_t nc = (uint32_t)__vimax_s32_relu(hi - lo + 1, 0);
            st.cells += nc;
            if (ZON) st.dc[PAR] = nc;
        }

        // (e) bases for antidiagonal e
        if (PAR == 1) {  // i advances: A fields move down one slot
            uint32_t in = 0;
            if (G > 1) in = __shfl_down_sync(gmask, Aw[0], 1, G) & FM;
            const uint32_t x = RF::fa(st.sa.next_fast(RF::SA));
            if (gl == G - 1) in = x;
            shift_down(Aw, in);
        } else {         // j advances: B fields move up one slot
            uint32_t in = 0;
            if (G > 1) in = __shfl_up_sync(gmask, top_field(Bw), 1, G);
            const uint32_t x = RF::fb(st.sb.next_fast(RF::SB));
            if (gl == 0) in = x;
            shift_up(Bw, in);
        }

        // (f) raw cells of e, relative to T_{e-1}: up / left from killed e-1,
        //     diag from killed e-2 rebased by -(T_{e-1} - T_{e-2}) = -dl
        const int32_t gp = P.gap;
        const int32_t sma = P.match - dl;
        const int32_t smi = P.mismatch - dl;
        const int32_t fg = DEAD - gp;  // max(up, left, fg) + gp >= DEAD: the floor
        constexpr bool SUB = fmt_base(FMT) == FMT_U8S;
        const int32_t sr = -dl;        // diagonal rebase (SUB: s' = table entry + sr)
        uint32_t X[NW];
#pragma unroll
        for (int q = 0; q < NW; ++q) X[q] = SUB ? Aw[q] + Bw[q] : Aw[q] ^ Bw[q];  // SUB: two table indices
        if (PAR == 1) {  // odd e: up = E[s+1], left = E[s], diag = O[s]
            int32_t nb = DEAD;  // E[R] of this lane = E[0] of the next lane
            if (G > 1) {
                nb = __shfl_down_sync(gmask, E[0], 1, G);
                if (gl == G - 1) nb = DEAD;
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int32_t up = (r < R - 1) ? E[r + 1] : nb;
                if (SUB) {
                    O[r] = cell_s(up, E[r], O[r], tab[(X[r / FPW] >> (CB * (r % FPW))) & FM], gp, fg, sr);
                } else {
                    const bool mis = ((X[r / FPW] >> (CB * (r % FPW))) & FM) != 0;
                    O[r] = cell(up, E[r], O[r], mis, gp, fg, sma, smi, P.one);
                }
            }
        } else {         // even e: up = O[s], left = O[s-1], diag = E[s]
            int32_t nb = DEAD;  // O[-1] of this lane = O[R-1] of the previous lane
            if (G > 1) {
                nb = __shfl_up_sync(gmask, O[R - 1], 1, G);
                if (gl == 0) nb = DEAD;
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int32_t left = (r > 0) ? O[r - 1] : nb;
                if (SUB) {
                    E[r] = cell_s(O[r], left, E[r], tab[(X[r / FPW] >> (CB * (r % FPW))) & FM], gp, fg, sr);
                } else {
                    const bool mis = ((X[r / FPW] >> (CB * (r % FPW))) & FM) != 0;
                    E[r] = cell(O[r], left, E[r], mis, gp, fg, sma, smi, P.one);
                }
            }
        }

        // (g) the maximum of raw e (key u' * KEYMUL + 1023 - slot), pending until
        //     step e + 2; any raw value above best_{e-1} is live (it is >= T_e)
        int32_t kq[NCH];
#pragma unroll
        for (int r = R - 1; r >= 0; --r) {
            const int32_t key = (PAR ? O[r] : E[r]) * KEYMUL + (1023 - r);
            const int c = r / RQ;
            const bool top = (r == R - 1) || (r == (c + 1) * RQ - 1);
            kq[c] = top ? key : max(kq[c], key);
        }
        int32_t kmax = kq[0];
#pragma unroll
        for (int c = 1; c < NCH; ++c)
            if (c * RQ < R) kmax = max(kmax, kq[c]);
        kmax -= gl * R;  // key = u' * KEYMUL + 1023 - (gl * R + r)
        // Z-drop (c-amb-19) needs the max over in-matrix cells only: cells past
        // the matrix stay below an earlier best (harmless for best) but can top
        // an antidiagonal; near the matrix edges the key is recomputed masked
        int32_t kz = kmax;
        if (ZON && P.zdrop >= 0) {
            const int32_t ch = (e + 1) >> 1, fh = e >> 1;
            const int32_t vlo = fh - st.n, vhi = st.m - ch;
            const int32_t base = st.S0 + gl * R;
            if (vlo > base || vhi < base + R - 1) {
                kz = INT32_MIN / 2;  // no valid slot (the offset below must not wrap)
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int32_t s = base + r;
                    if (s >= vlo && s <= vhi) kz = max(kz, (PAR ? O[r] : E[r]) * KEYMUL + (1023 - r));
                }
                kz -= gl * R;
            }
        }
        if (G > 1) {
            kmax = grp_max<G>(kmax, gmask);
            if (ZON && P.zdrop >= 0) kz = grp_max<G>(kz, gmask);
        }
        st.K[PAR] = kmax;
        if (ZON) st.KZ[PAR] = kz;
        st.d = e;
        return 0;
    }

    // window slot base S0 += 1 (band drifted towards higher slots); the pending
    // raw maximum of antidiagonal d (keys count slots from S0) moves with it
    __device__ __forceinline__ void shift_right(const Params &P, int32_t d) {
        int32_t eIn = DEAD, oIn = DEAD;
        uint32_t aIn = 0, bIn = 0;
        if (G > 1) {
            eIn = __shfl_down_sync(gmask, E[0], 1, G);
            oIn = __shfl_down_sync(gmask, O[0], 1, G);
            aIn = __shfl_down_sync(gmask, Aw[0], 1, G) & FM;
            bIn = __shfl_down_sync(gmask, Bw[0], 1, G) & FM;
        }
        const int32_t S1 = st.S0 + 1;
        if (gl == G - 1) {
            eIn = DEAD;
            oIn = DEAD;
            aIn = RF::fa(st.sa.next(P, RF::SA));  // a_{S1 + W - 1 + ceil(d/2)}
            bIn = RF::fb(seq_at<FMT>(P, st.sb.s, floor_half(d) - S1 - (W - 1), RF::SB));
        }
        if (gl == 0) st.sb.seek(P, st.sb.idx - 1);  // b stream steps back one base
        // rotate E/O through this thread's shared-memory slice: the reloads land in
        // the registers the arrays already occupy, so the common (no-shift) path
        // carries no register copies
        spill(E, O);
#pragma unroll
        for (int r = 0; r < R - 1; ++r) { E[r] = sbuf()[r + 1]; O[r] = sbuf()[R + r + 1]; }
        E[R - 1] = eIn;
        O[R - 1] = oIn;
        shift_down(Aw, aIn);
        shift_down(Bw, bIn);
        st.S0 = S1;
        adjust_pending(d, +1);
        ++st.shifts;
    }

    // window slot base S0 -= 1
    __device__ __forceinline__ void shift_left(const Params &P, int32_t d) {
        int32_t eIn = DEAD, oIn = DEAD;
        uint32_t aIn = 0, bIn = 0;
        if (G > 1) {
            eIn = __shfl_up_sync(gmask, E[R - 1], 1, G);
            oIn = __shfl_up_sync(gmask, O[R - 1], 1, G);
            aIn = __shfl_up_sync(gmask, top_field(Aw), 1, G);
            bIn = __shfl_up_sync(gmask, top_field(Bw), 1, G);
        }
        const int32_t S1 = st.S0 - 1;
        if (gl == 0) {
            eIn = DEAD;
            oIn = DEAD;
            aIn = RF::fa(seq_at<FMT>(P, st.sa.s, S1 + ceil_half(d), RF::SA));
            bIn = RF::fb(st.sb.next(P, RF::SB));  // b_{floor(d/2) - S1}
        }
        if (gl == G - 1) st.sa.seek(P, st.sa.idx - 1);  // a stream steps back one base
        spill(E, O);
#pragma unroll
        for (int r = 1; r < R; ++r) { E[r] = sbuf()[r - 1]; O[r] = sbuf()[R + r - 1]; }
        E[0] = eIn;
        O[0] = oIn;
        shift_up(Aw, aIn);
        shift_up(Bw, bIn);
        st.S0 = S1;
        adjust_pending(d, -1);
        ++st.shifts;
    }

    // The raw maximum of antidiagonal d (parity d&1) is still pending at a shift:
    // a slot index s becomes s - by, so the key's 1023 - s part grows by `by`.
    // (A raising maximum is a live cell inside the band, so it stays in 0..W-1;
    // a non-raising one is never decoded.)
    __device__ __forceinline__ void adjust_pending(int32_t d, int32_t by) {
        const bool p = d & 1;
        const int32_t k = p ? st.K[1] : st.K[0];
        const int32_t kn = k != KNONE ? k + by : k;
        st.K[0] = p ? st.K[0] : kn;
        st.K[1] = p ? kn : st.K[1];
        if (ZON) {
            const int32_t z = p ? st.KZ[1] : st.KZ[0];
            const int32_t zn = z != KNONE ? z + by : z;
            st.KZ[0] = p ? st.KZ[0] : zn;
            st.KZ[1] = p ? zn : st.KZ[1];
        }
    }
};

// Runs one group's task loop. `fetch(pos&)` yields the next list position (or
// false when there is none); the loop starts or resumes that task, sweeps it to
// completion or hand-over, and writes the result / publishes the hand-over.
// gpu-scope relaxed load (a volatile load compiles to a system-scope strong one)
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Starts or resumes the next task of a group (false: none left). The hot loop
// below always starts with an odd antidiagonal (a task resumed after an odd one
// takes the even one here), so it has a single code path; `rc` returns the
// outcome of that step (0 = go on). (A function, not a lambda: the inliner must
// not outline it, or the window's register arrays would move to local memory.)
template <class Win, class Fetch>
__device__ __forceinline__ bool start_next(Win &w, const Params &P, const LevelIO &io, Fetch &fetch, int &rc) {
    rc = 0;
    uint32_t pos;
    if (!fetch(pos)) return false;
    const uint32_t task = io.list[pos];
    const uint32_t rec = io.in_recs ? io.in_recs[pos] : NO_REC;
    if (rec != NO_REC) w.resume(P, io.rec_in + (size_t)rec * io.rec_in_stride);
    else w.init(P, task);
    if (io.stats && w.gl == 0) {
        atomicAdd((unsigned long long *)&io.stats->tasks_started[io.level], 1ull);
        if (io.is_helper) atomicAdd((unsigned long long *)&io.stats->helper_tasks, 1ull);
    }
    if (w.st.d & 1) rc = w.template step<0>(P, false);
    return true;
}

template <class Win, class Fetch>
__device__ __forceinline__ void run_group(Win &w, const Params &P, const LevelIO &io, Fetch fetch) {
    constexpr int G = Win::GG;
    const int lane = threadIdx.x & 31;
    const int leader = lane - w.gl;
    int rc = 0;
    bool active = start_next(w, P, io, fetch, rc);
    int32_t since = 0;  // antidiagonals at this level (hand-over test knob)
    while (active) {
        // one iteration = the odd then the even antidiagonal
        if (rc == 0) {
            // test knob (uniform, off in production): hand over at the next check point
            const bool force = io.handover > 0 && io.rec_out && since >= io.handover;
            rc = w.template step<1>(P, force);
            if (rc == 0) rc = w.template step<0>(P, false);
            since += 2;
        }
        if (rc != 0) {
            uint32_t rec = NO_REC;
            if (rc == 2 && io.rec_out) {  // hand the exact state to the next level
                if (w.gl == 0) {
                    rec = atomicAdd(io.rec_out_count, 1u);
                    if (rec >= io.rec_out_cap) rec = NO_REC;  // pool full: the next level restarts it
                }
                if (G > 1) rec = __shfl_sync(w.gmask, rec, leader);
                if (rec != NO_REC) w.save(P, io.rec_out + (size_t)rec * io.rec_out_stride);
                if (G > 1) __syncwarp(w.gmask);
            }
            if (rc == 1) w.finalize();
            if (w.gl == 0) {
                if (rc == 1) {
                    TaskRes tr;
                    tr.best = w.st.best;
                    tr.i = w.st.arg_i;
                    tr.j = w.st.arg_j;
                    tr.flags = 0;
                    tr.cells = w.st.cells;
                    io.tres[w.st.task] = tr;
                } else {
                    // publish: record index first, then the task id (the entry's
                    // ready flag for in-kernel consumers; lists start as NO_TASK)
                    const uint32_t o = atomicAdd(io.out_count, 1u);
                    if (io.out_recs) io.out_recs[o] = rec;
                    __threadfence();
                    *(volatile uint32_t *)&io.out_list[o] = w.st.task;
                }
                if (io.stats) {
                    atomicAdd((unsigned long long *)&io.stats->window_shifts, (unsigned long long)w.st.shifts);
                    if (rc == 1)
                        atomicAdd((unsigned long long *)&io.stats->tasks_finished[io.level], 1ull);
                    if (rc == 1 || rec != NO_REC) {
                        atomicAdd((unsigned long long *)&io.stats->cells_per_level[io.level],
                                  (unsigned long long)(w.st.cells - w.st.cells_entry));
                    }
                    if (rc == 1) atomicAdd((unsigned long long *)&io.stats->cells_total, (unsigned long long)w.st.cells);
                }
            }
            if (rc == 2) w.st.shifts = 0;
            since = 0;
            active = start_next(w, P, io, fetch, rc);
        }
    }
}


// Persistent kernel: each group of G lanes pulls tasks from the level's list.
// A level may exist in two shapes (throughput: G small, R = 32; latency: one
// warp per task); the launch whose [min_count, max_count) holds the list length
// runs, the other exits at once (no host synchronisation).
//
// With HR > 0 (first level only), the last warp of the first `io.helpers`
// blocks runs the NEXT level in its latency shape (one warp per task, window
// 32*HR) on the tasks this level hands over, as soon as each is published:
// overflowing tasks then finish while this level is still running instead of
// forming a serial tail after it. What the helpers do not take, the next
// level's own launch does (it shares their cursor).
template <int G, int R, int FMT, bool M2> struct Window16;  // xdrop_window16.cuh

// PK: 0 = the producers run the int32 window (Window), 1 = the packed int16
// window (Window16), 2 = the packed window specialised for match - mismatch = 2
template <int G, int R, int FMT, int HG, int HR, int PK = 0>
__global__ void __launch_bounds__(128, (PK ? (G == 1 ? (R <= 24 ? 4 : LOGAN_PK_MINB) : 3)
                                           : (G == 1 ? ((fmt_z(FMT) || fmt_base(FMT) == FMT_U8S) ? 3 : LOGAN_L0_MINB) : 1)))
    k_window(const Params P, const LevelIO io, const LevelIO hio) {
    using PW = typename std::conditional<(PK != 0), Window16<G, R, FMT, PK == 2>, Window<G, R, FMT>>::type;
    const uint32_t count = *io.count;
    const uint32_t taken = *io.cursor;  // entries already taken (by in-kernel helpers)
    const uint32_t remaining = count - (taken < count ? taken : count);
    if (remaining < io.min_count || remaining >= io.max_count) return;
    extern __shared__ int32_t win_smem[];
    const int lane = threadIdx.x & 31;
    int8_t *tab = nullptr;
    if (fmt_base(FMT) == FMT_U8S) {  // the substitution table behind the per-thread shift slices
        constexpr int S1 = Window<G, R, FMT>::SB_STRIDE;
        constexpr int S2 = HR > 0 ? Window<(HG > 0 ? HG : 32), (HR > 0 ? HR : 1), FMT>::SB_STRIDE : 0;
        tab = (int8_t *)(win_smem + blockDim.x * (S1 > S2 ? S1 : S2));
        load_subst_tab(P, tab, threadIdx.x, blockDim.x);
        __syncthreads();
    }
    // helpers: the warp that takes the LAST wave of the static first round (below)
    // in the LAST io.helpers blocks, so the producers' static chunks are dense
    const int hwarp = (io.sms > 0 && ((gridDim.x / (uint32_t)io.sms) & 1) == 0) ? 0 : (int)(blockDim.x >> 5) - 1;
    const bool helper = HR > 0 && (int)blockIdx.x >= (int)gridDim.x - io.helpers && (int)(threadIdx.x >> 5) == hwarp;
    if (HR > 0 && helper) {
        constexpr int HG_ = HG > 0 ? HG : 32, HR_ = HR > 0 ? HR : 1;
        // packed producers get packed helpers (the same int16 window one width up):
        // a task that overflows late in its life finishes at the packed rate
        constexpr bool HPK = PK != 0 && HR_ >= 16 && HR_ % 4 == 0;
        using HW = typename std::conditional<HPK, Window16<HG_, HR_, FMT, PK == 2>, Window<HG_, HR_, FMT>>::type;
        HW w;
        w.tab = tab;
        w.sbase = win_smem + threadIdx.x * HW::SB_STRIDE;
        w.gl = lane % HG_;
        w.gmask = (HG_ == 32) ? 0xffffffffu : (((1u << HG_) - 1u) << (lane - w.gl));
        const int leader = lane - w.gl;
        const uint32_t total = io.workers;
        // Helpers only work while producers are still sweeping: once every
        // producer group is done they stop taking entries, and whatever is left
        // goes to the next level's own launch (throughput shape if many).
        auto fetch = [&](uint32_t &pos) -> bool {
            // take a new entry only while producers are running; idle helpers back
            // off (their polls would take issue slots from the producers on their SM)
            for (uint32_t ns = 256;; ns = ns < 4096 ? 2 * ns : ns) {
                if (ld_relaxed(io.done) == total) return false;
                if (ld_relaxed(hio.cursor) < ld_relaxed(io.out_count)) break;
                __nanosleep(ns);
            }
            uint32_t p = 0;
            if (w.gl == 0) p = atomicAdd(hio.cursor, 1u);
            if (HG_ > 1) p = __shfl_sync(w.gmask, p, leader);
            // a claimed position is either processed here or proven not to exist
            for (;;) {
                if (p < ld_relaxed(io.out_count)) break;
                if (ld_relaxed(io.done) == total) {
                    __threadfence();
                    if (p >= ld_relaxed(io.out_count)) return false;
                    break;
                }
                __nanosleep(500);
            }
            while (ld_relaxed(&io.out_list[p]) == NO_TASK) __nanosleep(64);
            __threadfence();
            pos = p;
            return true;
        };
        run_group(w, P, hio, fetch);
        return;
    }
    PW w;
    w.tab = tab;
    w.sbase = win_smem + threadIdx.x * PW::SB_STRIDE;
    w.gl = lane % G;
    w.gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - w.gl));
    const int leader = lane - w.gl;
    // First level (io.sms > 0): a static first round spreads the LPT queue's head
    // over the SM sub-partitions. With blocks dispatched round-robin (block b on SM
    // s = b mod #SM, block row r = b div #SM, warp w on sub-partition w), chunk
    // c = s + #SM * k takes wave k = 4 r + (r even ? w : 3 - w) (32 / G tasks per
    // warp): the longest #SM chunks go one per SM to sub-partition 0, the next to
    // 1, ..., and the rows run serpentine so every sub-partition gets a balanced
    // share of the long chunks -- what matters when the tasks are few (a
    // strong-scaling share), harmless when they are many. The helpers own the
    // last wave's last chunk numbers, so the producers' chunks are dense. Later
    // fetches take the dynamic cursor past the static region.
    const uint32_t wib = threadIdx.x >> 5;
    const uint32_t gpw = 32 / G;  // groups per warp
    const uint32_t nprod = gridDim.x * (blockDim.x >> 5) - (uint32_t)io.helpers;  // producer warps
    const bool stat = io.sms > 0 && (gridDim.x % (uint32_t)io.sms) == 0 && (blockDim.x >> 5) == 4;
    const uint32_t sbase = stat ? nprod * gpw : 0u;
    bool first = stat;
    auto fetch = [&](uint32_t &pos) -> bool {
        uint32_t p = 0xffffffffu;
        if (first) {
            first = false;
            const uint32_t r = blockIdx.x / io.sms;
            const uint32_t k = 4u * r + ((r & 1u) ? 3u - wib : wib);
            const uint32_t c = blockIdx.x % io.sms + io.sms * k;
            p = c * gpw + (uint32_t)(lane / G);
        } else {
            if (w.gl == 0) p = atomicAdd(io.cursor, 1u) + sbase;
            if (G > 1) p = __shfl_sync(w.gmask, p, leader);
        }
        pos = p;
        return p < count;
    };
    run_group(w, P, io, fetch);
    if (HR > 0 && w.gl == 0) {  // this group will publish no more hand-overs
        __threadfence();
        atomicAdd(io.done, 1u);
    }
}

}  // namespace logan
