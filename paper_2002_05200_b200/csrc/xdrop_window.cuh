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
//  * Scores are stored RELATIVE to the kill threshold T_d = best_{d-1} - X:
//    u = S - T_d, live <=> u >= 0. The per-step rebase folds into the two
//    scoring constants (gap' = gap - (T_d - T_{d-1}), s' = s - (T_d - T_{d-2}))
//    so the cell is three DPX VIADDMNMX plus one VIMNMX.U32:
//        u = max(max(up, left, DEAD - gap') + gap', diag + s');  u = min_u32(u, DEAD)
//    (VIMNMX3, an add, VIADDMNMX, VIMNMX.U32), which maps every negative u to
//    exactly DEAD = -2^20 (an exact, absorbing kill: a dead value can never
//    climb back within 2^20 / match steps, far more than any task's
//    antidiagonal count at the ABI's limits).
//  * Bases sit in registers, 4-bit fields (2-bit pool) or 16-bit fields (u8
//    pool), one per slot; positions past an extension's end hold sentinels
//    that match nothing, so cells outside the matrix (i > m or j > n) can only
//    hold values below an earlier best and are excluded from the band
//    bookkeeping by a per-lane validity mask -- no per-cell masking.
//  * Per antidiagonal the max and its slot come from one packed key
//    (u * 1027 + 1023 - slot, an IMAD) reduced with VIMNMX3 inside the lane and SHFL
//    butterflies across the G lanes; the live extremes from a funnel-shifted
//    sign mask + FLO. Ties go to the smallest slot = smallest i (c-amb-9).
//  * The window re-centres by one slot when the band touches an edge; if the
//    band is wider than W - 2 slots the task is handed to the next level.
#pragma once

#include "xdrop_common.cuh"

namespace logan {

constexpr int32_t DEAD = -(1 << 20);
constexpr uint32_t DEADU = 0xFFF00000u;  // (uint32_t)DEAD
// Argmax key of a cell: u * KEYMUL + (1023 - slot). KEYMUL > 1023 keeps the
// order (value, then smallest slot); it is not a power of two so the key is
// one IMAD on the FMA pipe (the ALU pipe is the kernel's bottleneck).
// |DEAD| * KEYMUL < 2^31 and (X + 2*127) * KEYMUL < 2^31 for X <= 2^19.
constexpr int32_t KEYMUL = 1027;

// How many of the 4 sign-mask chains run on the FMA pipe (the rest use SHF on
// the ALU pipe): balances the two pipes (tuned by measurement).
// Minimum resident blocks per SM requested for the one-lane-per-task kernels
// (caps registers; tuned by measurement).
#ifndef LOGAN_L0_MINB
#define LOGAN_L0_MINB 1
#endif

#ifndef LOGAN_NCHAIN
#define LOGAN_NCHAIN 4
#endif

#ifndef LOGAN_MASK_FMA_CHAINS
#define LOGAN_MASK_FMA_CHAINS 0
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

// Group-uniform state of one task (replicated in each lane of the group).
template <int FMT>
struct WinState {
    // sa feeds the top slot (read by lane G-1; sa.idx = S0 + W + ceil(d/2)),
    // sb feeds the bottom slot (read by lane 0; sb.idx = floor(d/2) - S0 + 1)
    Stream<FMT> sa, sb;
    uint32_t task;
    int32_t m, n;
    int32_t d;             // last antidiagonal computed
    int32_t S0;            // slot of the window's first register
    int32_t best, arg_i, arg_j;
    // thresholds: Tn = T_{d+1}; Tq[p] = the last T_e with e of parity p
    // (after antidiagonal d: Tq[d&1] = T_d, Tq[(d-1)&1] = T_{d-1}). Indexing by
    // parity (a compile-time constant inside a step) means nothing rotates.
    int32_t Tn, Tq[2];
    // live slot extremes of the last antidiagonal of each parity (sF[d&1] is
    // antidiagonal d, sF[(d-1)&1] is d-1); an antidiagonal without a (valid)
    // live cell has sF = EMPTY_F, sL = EMPTY_L, which makes every min / max
    // below ignore it without a branch
    int32_t sF[2], sL[2];
    uint64_t cells;
    uint64_t cells_entry;  // cells already counted when the task entered this level
    uint32_t shifts;
};

// Hand-over record between levels: REC_HDR ints of scalars, then E[W], O[W].
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
    static_assert(R >= 1 && R <= 32 && W <= 1024 && (G & (G - 1)) == 0, "window shape");

    int32_t E[R], O[R];
    uint32_t Aw[NW], Bw[NW];
    WinState<FMT> st;
    int gl;            // lane within group
    unsigned gmask;

    // One cell (eq. P:85 + the drop rule P:89) on threshold-relative values:
    //   u = max(max(up, left, fg) + gap', diag + s'), then the exact kill
    //   min_u32(u, DEAD): every negative u becomes DEAD, live values stay.
    // The kernel is bound by the ALU pipe (VIMNMX3, VIADDMNMX, VIMNMX.U32 and
    // the mismatch test live there), so diag + s' is computed on the FMA pipe:
    // an IMAD by an opaque run-time 1 for the match case, overwritten by a
    // predicated IMAD for a mismatch -- no SEL, no IADD3.
    // Substitution-matrix cell: s = the table entry, sr = the diagonal rebase.
    __device__ __forceinline__ static int32_t cell_s(int32_t up, int32_t left, int32_t diag, int32_t s,
                                                     int32_t gp, int32_t fg, int32_t sr) {
        const int32_t t0 = __vimax3_s32(up, left, fg);
        const int32_t u = __viaddmax_s32(t0, gp, diag + s + sr);
        return (int32_t)min((uint32_t)u, DEADU);
    }
    const int8_t *tab;  // FMT_U8S: the substitution table in shared memory

    __device__ __forceinline__ static int32_t cell(int32_t up, int32_t left, int32_t diag, bool mis,
                                                   int32_t gp, int32_t fg, int32_t sma, int32_t smi,
                                                   int32_t one) {
        const int32_t t0 = __vimax3_s32(up, left, fg);
        int32_t dps;
        asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(dps) : "r"(diag), "r"(one), "r"(sma));
        asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q mad.lo.s32 %0, %2, %3, %4;\n\t}"
            : "+r"(dps) : "r"((uint32_t)mis), "r"(diag), "r"(one), "r"(smi));
        const int32_t u = __viaddmax_s32(t0, gp, dps);
        return (int32_t)min((uint32_t)u, DEADU);
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
        w[0] = (NW == 1 ? (w[0] << CB) : (w[0] << CB)) | in;
        if (RL < FPW) w[NW - 1] &= (1u << (CB * RL)) - 1u;
    }

    // ---- task start -----------------------------------------------------------
    __device__ __forceinline__ void init(const Params &P, uint32_t task) {
        const TaskDesc td = task_desc(P, task);
        st.task = task;
        st.m = td.a.len;
        st.n = td.b.len;
        st.d = 0;
        st.S0 = -(W / 2);
        st.best = 0;
        st.arg_i = st.arg_j = 0;
        st.Tq[0] = -P.xdrop;  // T_0 = best_{-1} - X with best_{-1} := 0
        st.Tq[1] = -P.xdrop;  // T_{-1}
        st.Tn = -P.xdrop;     // T_1 = best_0 - X
        st.sF[0] = st.sL[0] = 0;  // antidiagonal 0: the origin (slot 0)
        st.sF[1] = EMPTY_F;       // antidiagonal -1: empty
        st.sL[1] = EMPTY_L;
        st.cells = 0;
        st.shifts = 0;
        // values: origin S(0,0) = 0 -> u = 0 - T_0 = X; everything else dead
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

    // ---- exact hand-over between levels ---------------------------------------
    // A task whose band outgrows this window is written out after antidiagonal
    // d (values of d and d-1 plus every scalar) and the next, wider level
    // continues it from d + 1: cells outside the old window are dead (the band
    // invariant), so the continuation is exact.
    __device__ __forceinline__ void save(int32_t *rec) const {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            rec[REC_HDR + gl * R + r] = E[r];
            rec[REC_HDR + W + gl * R + r] = O[r];
        }
        if (gl == 0) {
            rec[0] = (int32_t)st.task; rec[1] = st.d; rec[2] = st.S0; rec[3] = st.best;
            const bool odd = st.d & 1;  // record order: d, then d-1
            rec[4] = st.arg_i; rec[5] = st.arg_j; rec[6] = st.Tn;
            rec[7] = odd ? st.Tq[1] : st.Tq[0];
            rec[8] = odd ? st.Tq[0] : st.Tq[1];
            rec[9] = odd ? st.sF[1] : st.sF[0];
            rec[10] = odd ? st.sL[1] : st.sL[0];
            rec[11] = odd ? st.sF[0] : st.sF[1];
            rec[12] = odd ? st.sL[0] : st.sL[1];
            rec[13] = 0;
            rec[14] = (int32_t)st.shifts; rec[15] = W;
            rec[16] = (int32_t)(uint32_t)st.cells; rec[17] = (int32_t)(uint32_t)(st.cells >> 32);
        }
    }

    __device__ __forceinline__ void resume(const Params &P, const int32_t *rec) {
        st.task = (uint32_t)rec[0];
        const TaskDesc td = task_desc(P, st.task);
        st.m = td.a.len;
        st.n = td.b.len;
        st.sa.s = td.a;
        st.sb.s = td.b;
        st.d = rec[1];
        const int32_t S0src = rec[2];
        st.best = rec[3]; st.arg_i = rec[4]; st.arg_j = rec[5];
        const bool odd = st.d & 1;
        st.Tn = rec[6];
        st.Tq[0] = odd ? rec[8] : rec[7];
        st.Tq[1] = odd ? rec[7] : rec[8];
        st.sF[0] = odd ? rec[11] : rec[9];
        st.sF[1] = odd ? rec[9] : rec[11];
        st.sL[0] = odd ? rec[12] : rec[10];
        st.sL[1] = odd ? rec[10] : rec[12];
        st.shifts = (uint32_t)rec[14];
        const int32_t Wsrc = rec[15];
        st.cells = (uint64_t)(uint32_t)rec[16] | ((uint64_t)(uint32_t)rec[17] << 32);
        st.cells_entry = st.cells;
        // centre the wider window on the live band of d and d-1
        int32_t Fm = min(st.sF[0], st.sF[1]), Lm = max(st.sL[0], st.sL[1]);
        if (Fm > Lm) { Fm = S0src; Lm = S0src + Wsrc - 1; }
        st.S0 = ((Fm + Lm) >> 1) - W / 2;
        const int32_t s0 = st.S0 + gl * R;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int32_t q = s0 + r - S0src;
            const bool in = q >= 0 && q < Wsrc;
            E[r] = in ? rec[REC_HDR + q] : DEAD;
            O[r] = in ? rec[REC_HDR + Wsrc + q] : DEAD;
        }
        load_bases(P);
    }

    // ---- one antidiagonal d = st.d + 1 of parity PAR ---------------------------
    // returns 0 = continue, 1 = finished, 2 = overflow
    template <int PAR>
    __device__ __forceinline__ int step(const Params &P) {
        const int32_t d = st.d + 1;
        const int32_t ch = PAR ? (d + 1) >> 1 : d >> 1, fh = PAR ? (d - 1) >> 1 : d >> 1;

        // (1) band cells of antidiagonal d from the live extremes of d-1, d-2
        //     (c-amb-14: lo = max(1, d-n, min(F1, F2+1)), hi = min(m, d-1, max(L1, L2)+1))
        //     Empty antidiagonals carry EMPTY_F / EMPTY_L and drop out of the
        //     min / max; d = 1 clips to an empty band by itself.
        {
            // column of slot 0 on d-1 (c1) and d-2 (c2 = c1 - 1 + PAR), so with
            // c = c1: odd d: lo = max(min(F1, F2 + 1) + c, 1, d-n), hi = min(max(L1, L2) + c + 1, m, d-1);
            // even d: lo = max(min(F1, F2) + c, 1, d-n), hi = min(max(L1, L2 - 1) + c + 1, m, d-1)
            // (3-input DPX min / max; d-1 has the other parity, d-2 this parity)
            const int32_t c = PAR ? (d - 1) >> 1 : d >> 1;
            const int32_t F1 = st.sF[1 - PAR], F2 = st.sF[PAR], L1 = st.sL[1 - PAR], L2 = st.sL[PAR];
            const int32_t fmin = PAR ? min(F1, F2 + 1) : min(F1, F2);
            const int32_t lmax = PAR ? max(L1, L2) : max(L1, L2 - 1);
            const int32_t lo = __vimax3_s32(fmin + c, 1, d - st.n);
            const int32_t hi = __vimin3_s32(lmax + c + 1, st.m, d - 1);
            st.cells += (uint32_t)__vimax_s32_relu(hi - lo + 1, 0);
        }

        // (2) bases for antidiagonal d
        if (PAR == 1) {  // i advances: A fields move down one slot
            uint32_t in = 0;
            if (G > 1) in = __shfl_down_sync(gmask, Aw[0], 1, G) & FM;
            // one or two lanes per task: many lanes of the warp read a stream, so its
            // refill is predicated; wider groups have few readers per warp: branch
            if (gl == G - 1) in = RF::fa(G <= 2 ? st.sa.next_fast(RF::SA) : st.sa.next(P, RF::SA));
            shift_down(Aw, in);
        } else {         // j advances: B fields move up one slot
            uint32_t in = 0;
            if (G > 1) in = __shfl_up_sync(gmask, top_field(Bw), 1, G);
            if (gl == 0) in = RF::fb(G <= 2 ? st.sb.next_fast(RF::SB) : st.sb.next(P, RF::SB));
            shift_up(Bw, in);
        }

        // (3) rebased constants (T_d = st.Tn is this step's threshold; T_{d-1} is
        //     the other parity's, T_{d-2} this parity's)
        const int32_t Tc = st.Tn;
        const int32_t gp = P.gap - (Tc - st.Tq[1 - PAR]);
        const int32_t sma = P.match - (Tc - st.Tq[PAR]);
        const int32_t smi = P.mismatch - (Tc - st.Tq[PAR]);
        const int32_t fg = DEAD - gp;  // max(up, left, fg) + gp >= DEAD: the floor

        const uint32_t two = 2u * (uint32_t)P.one;  // = 2, opaque to the compiler
        constexpr bool SUB = fmt_base(FMT) == FMT_U8S;
        const int32_t sr = -(Tc - st.Tq[PAR]);  // diagonal rebase (SUB: s' = table entry + sr)
        uint32_t X[NW];
#pragma unroll
        for (int q = 0; q < NW; ++q) X[q] = SUB ? Aw[q] + Bw[q] : Aw[q] ^ Bw[q];  // SUB: two table indices

        // (4) cells
        constexpr int NCH = LOGAN_NCHAIN;  // independent key / dead-mask chains per lane
        int32_t kq[NCH];
        uint32_t dq[NCH];
        constexpr int RQ = (R + NCH - 1) / NCH;
        if (PAR == 1) {
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
        } else {
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
        // keys u * KEYMUL + 1023 - r and dead masks over the new antidiagonal
#pragma unroll
        for (int r = R - 1; r >= 0; --r) {
            const int32_t u = PAR ? O[r] : E[r];
            const int c = r / RQ;
            const bool top = (r == R - 1) || (r == (c + 1) * RQ - 1);  // first slot of chain c
            const int32_t key = u * KEYMUL + (1023 - r);
            kq[c] = top ? key : max(kq[c], key);
            if (LOGAN_MASK_FMA_CHAINS > c) {  // two IMADs on the FMA pipe
                // append sign(u) (1 = dead) as bit (r - c*RQ): dq = 2*dq + (u >>> 31)
                uint32_t sg;
                asm("mul.hi.u32 %0, %1, %2;" : "=r"(sg) : "r"((uint32_t)u), "r"(two));
                if (top) dq[c] = sg;
                else asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(dq[c]) : "r"(dq[c]), "r"(two), "r"(sg));
            } else {  // one funnel shift on the ALU pipe (same bit order)
                dq[c] = top ? ((uint32_t)u >> 31) : __funnelshift_l((uint32_t)u, dq[c], 1);
            }
        }
        int32_t kmax = kq[0];
#pragma unroll
        for (int c = 1; c < NCH; ++c)
            if (c * RQ < R) kmax = max(kmax, kq[c]);
        uint32_t dead = 0;
#pragma unroll
        for (int c = 0; c < NCH; ++c)
            if (c * RQ < R) dead |= dq[c] << (c * RQ);

        // (5) validity of slots for this lane: cells with i < 0 or j < 0 are dead
        //     by construction; cells past the matrix (i > m or j > n) are masked
        //     out of the band bookkeeping (slot s: i <= m <=> s <= m - ch,
        //     j <= n <=> s >= fh - n). Most steps take the all-valid path.
        const int32_t vlo = fh - st.n, vhi = st.m - ch;
        const int32_t base = st.S0 + gl * R;
        uint32_t vmask = (R == 32) ? 0xffffffffu : ((1u << R) - 1u);
        if (vlo > base || vhi < base + R - 1) {
            const int32_t rlo = max(vlo - base, 0), rhi = min(vhi - base, R - 1);
            vmask = (rlo <= rhi) ? ((0xffffffffu >> (31 - rhi)) & ~((1u << rlo) - 1u)) : 0u;
        }
        const uint32_t live = ~dead & vmask;
        // one lane per task: the extremes are only read when live != 0, so no
        // sentinel selects (a sub-warp or warp group reduces with sentinels)
        int32_t lf = G == 1 ? __ffs(live) - 1 : (live ? gl * R + __ffs(live) - 1 : INT32_MAX);
        int32_t ll = G == 1 ? 31 - __clz(live) : (live ? gl * R + 31 - __clz(live) : INT32_MIN);
        kmax = kmax - gl * R;  // key = u*KEYMUL + 1023 - (gl*R + r)
        // Z-drop (c-amb-19) needs the max over in-matrix cells only: cells past
        // the matrix stay below an earlier best (harmless for best) but can top
        // an antidiagonal; near the matrix edges the key is recomputed masked
        int32_t kz = kmax;
        const bool zon = fmt_z(FMT) && P.zdrop >= 0;
        if (zon && vmask != ((R == 32) ? 0xffffffffu : ((1u << R) - 1u))) {
            kz = INT32_MIN / 2;  // no valid slot (the offset below must not wrap)
#pragma unroll
            for (int r = 0; r < R; ++r)
                if ((vmask >> r) & 1u) kz = max(kz, (PAR ? O[r] : E[r]) * KEYMUL + (1023 - r));
            kz -= gl * R;
        }
        if (G > 1) {
            kmax = grp_max<G>(kmax, gmask);
            lf = grp_min<G>(lf, gmask);
            ll = grp_max<G>(ll, gmask);
            if (zon) kz = grp_max<G>(kz, gmask);
        }
        const bool h = G == 1 ? live != 0 : (lf != INT32_MAX);

        // (6) best after the complete antidiagonal; argmax on strict increase
        // V = u + T_d > best_{d-1} = T_d + X  <=>  u > X  <=>  kmax >= (X + 1) * KEYMUL:
        // the key decode runs only on antidiagonals that raise best
        if (kmax >= (P.xdrop + 1) * KEYMUL) {
            const int32_t ku = kmax / KEYMUL;
            st.best = ku + Tc;
            const int32_t slot = st.S0 + (1023 - (kmax - ku * KEYMUL));
            st.arg_i = slot + ch;
            st.arg_j = d - st.arg_i;
        }
        // Z-drop stop (c-amb-19): best - M_d > Z + |gap| * |(i_d - i*) - (j_d - j*)|
        // Every live u is >= 0 and best >= T_d + X, so a stop needs u_max < X - Z on
        // this antidiagonal: key below (X - Z) * KEYMUL (cheap test first; an
        // antidiagonal that raised best has u_max > X and never stops)
        bool zstop = false;
        if (zon && kz >= 0 && kz < (P.xdrop - P.zdrop) * KEYMUL) {
            const int32_t kzu = kz / KEYMUL;
            const int32_t zi = st.S0 + (1023 - (kz - kzu * KEYMUL)) + ch;
            const int32_t off = abs((zi - st.arg_i) - ((d - zi) - st.arg_j));
            zstop = st.best - (kzu + Tc) > P.zdrop - P.gap * off;
        }
        st.Tq[PAR] = Tc;
        st.Tn = st.best - P.xdrop;
        st.d = d;

        st.sF[PAR] = h ? st.S0 + lf : EMPTY_F;
        st.sL[PAR] = h ? st.S0 + ll : EMPTY_L;
        // The checks below run after the even antidiagonal only. The band's
        // right edge can grow (by one slot) only on even steps and its left
        // edge only on odd steps, so the margin-1 invariant checked here keeps
        // every cell outside the window dead through both steps of the next
        // iteration. An odd antidiagonal that ends the task is followed by one
        // extra even one whose band is empty: no cells, no best change.
        if (PAR == 1) return zstop ? 1 : 0;

        // (7) termination: antidiagonals d and d-1 both empty (c-amb-7), or Z-drop
        if (zstop || (st.sF[0] == EMPTY_F && st.sF[1] == EMPTY_F)) return 1;

        // (8) keep the live band of d and d-1 inside [S0+1, S0+W-2]
        const int32_t Fm = min(st.sF[0], st.sF[1]), Lm = max(st.sL[0], st.sL[1]);
        const bool lowv = Fm < st.S0 + 1, highv = Lm > st.S0 + W - 2;
        if (lowv || highv) {
            if (lowv && highv) return 2;
            if (lowv) {
                if (Lm > st.S0 + W - 3) return 2;
                shift_left(P, d);
            } else {
                if (Fm < st.S0 + 2) return 2;
                shift_right(P, d);
            }
        }
        return 0;
    }

    // window slot base S0 += 1 (band drifted towards higher slots)
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
        ++st.shifts;
    }
};

// Runs one group's task loop. `fetch(pos&)` yields the next list position (or
// false when there is none); the loop starts or resumes that task, sweeps it to
// completion or hand-over, and writes the result / publishes the hand-over.
template <class Win, class Fetch>
__device__ __forceinline__ void run_group(Win &w, const Params &P, const LevelIO &io, Fetch fetch) {
    constexpr int G = Win::GG;
    const int lane = threadIdx.x & 31;
    const int leader = lane - w.gl;
    // start or resume the next task; a task resumed after an odd antidiagonal
    // takes the even one here, so the hot loop below always starts at an even d
    // (a single code path: no per-iteration register shuffling). `rc` returns
    // the outcome of that alignment step (0 = keep sweeping).
    auto next_task = [&](int &rc) -> bool {
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
        if (w.st.d & 1) rc = w.template step<0>(P);
        return true;
    };

    int rc = 0;
    bool active = next_task(rc);
    int32_t since = 0;  // antidiagonals at this level (hand-over test knob)
    while (active) {
        // one iteration = the odd then the even antidiagonal
        if (rc == 0) {
            rc = w.template step<1>(P);
            if (rc == 0) rc = w.template step<0>(P);
        }
        if (io.handover > 0) {  // test knob (uniform branch, off in production)
            since += 2;
            if (rc == 0 && io.rec_out && since >= io.handover) rc = 2;
        }
        if (rc != 0) {
            uint32_t rec = NO_REC;
            if (rc == 2 && io.rec_out) {  // hand the exact state to the next level
                if (w.gl == 0) {
                    rec = atomicAdd(io.rec_out_count, 1u);
                    if (rec >= io.rec_out_cap) rec = NO_REC;  // pool full: the next level restarts it
                }
                if (G > 1) rec = __shfl_sync(w.gmask, rec, leader);
                if (rec != NO_REC) w.save(io.rec_out + (size_t)rec * io.rec_out_stride);
                if (G > 1) __syncwarp(w.gmask);
            }
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
            active = next_task(rc);
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
template <int G, int R, int FMT, int HG, int HR>
__global__ void __launch_bounds__(128, (G == 1 ? ((fmt_z(FMT) || fmt_base(FMT) == FMT_U8S) ? 3 : LOGAN_L0_MINB) : 1))
    k_window(const Params P, const LevelIO io, const LevelIO hio) {
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
    const bool helper = HR > 0 && (int)blockIdx.x < io.helpers && (threadIdx.x >> 5) == (blockDim.x >> 5) - 1;
    if (HR > 0 && helper) {
        constexpr int HG_ = HG > 0 ? HG : 32, HR_ = HR > 0 ? HR : 1;
        Window<HG_, HR_, FMT> w;
        w.tab = tab;
        w.sbase = win_smem + threadIdx.x * Window<HG_, HR_, FMT>::SB_STRIDE;
        w.gl = lane % HG_;
        w.gmask = (HG_ == 32) ? 0xffffffffu : (((1u << HG_) - 1u) << (lane - w.gl));
        const int leader = lane - w.gl;
        const uint32_t total = io.workers;
        // Helpers only work while producers are still sweeping: once every
        // producer group is done they stop taking entries, and whatever is left
        // goes to the next level's own launch (throughput shape if many).
        auto fetch = [&](uint32_t &pos) -> bool {
            for (;;) {  // take a new entry only while producers are running
                if (*(volatile const uint32_t *)io.done == total) return false;
                if (*(volatile const uint32_t *)hio.cursor < *(volatile const uint32_t *)io.out_count) break;
                __nanosleep(1000);
            }
            uint32_t p = 0;
            if (w.gl == 0) p = atomicAdd(hio.cursor, 1u);
            if (HG_ > 1) p = __shfl_sync(w.gmask, p, leader);
            // a claimed position is either processed here or proven not to exist
            for (;;) {
                if (p < *(volatile const uint32_t *)io.out_count) break;
                if (*(volatile const uint32_t *)io.done == total) {
                    __threadfence();
                    if (p >= *(volatile const uint32_t *)io.out_count) return false;
                    break;
                }
                __nanosleep(500);
            }
            while (*(volatile const uint32_t *)&io.out_list[p] == NO_TASK) __nanosleep(64);
            __threadfence();
            pos = p;
            return true;
        };
        run_group(w, P, hio, fetch);
        return;
    }
    Window<G, R, FMT> w;
    w.tab = tab;
    w.sbase = win_smem + threadIdx.x * Window<G, R, FMT>::SB_STRIDE;
    w.gl = lane % G;
    w.gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - w.gl));
    const int leader = lane - w.gl;
    auto fetch = [&](uint32_t &pos) -> bool {
        uint32_t p = 0xffffffffu;
        if (w.gl == 0) p = atomicAdd(io.cursor, 1u);
        if (G > 1) p = __shfl_sync(w.gmask, p, leader);
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
