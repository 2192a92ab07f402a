// xdrop_window16.cuh — register windows with PACKED int16 pairs: G lanes per
// task, R slots per lane (R in {16, 20, 24, 28, 32}), W = G * R, 2-bit pools,
// X <= 16000. The first level (G = 1) and the throughput shapes of levels 2-5
// (G = W / 32, R = 32) and the wide latency shapes (one warp, R >= 16). The
// sweep is the one of xdrop_window.cuh (same method citations, same pipelined
// "kill one antidiagonal late" state, same hand-over records); only the
// per-slot arithmetic differs.
//
// Why: the int32 window is bound by instruction issue (~88
// thread-instructions per SM clock, the practical limit measured by
// tools/int_peak.cu) and the ALU pipe (~80%). Two slots per DPX instruction
// (VIMNMX3.S16x2, VIADDMNMX.S16x2, VIADDMNMX.U16x2; VIADD.16x2 issues on the
// FMA side) about halves the instructions per slot.
//
// Layout ("split pairs"): word k of a lane's E / O holds its slot k in the low
// half and slot k + H in the high half (H = R/2). Slot s's neighbours s+1 and
// s-1 are then the next / previous WORD (both halves move together), so a cell
// pair needs no realignment, except at the one seam word per step (one PRMT,
// with one SHFL from the neighbouring lane when G > 1).
// Values are int16 relative to the thresholds (live u <= X + 3*127 < 2^15,
// DEAD16 = -16384, dead values stay in [DEAD16 - 3*127, DEAD16]).
//
// Substitution per pair: the 4-bit base fields hold 3-bit codes (bases 0..3,
// past-the-end sentinels 4 for A and 5 for B, so every XOR of two fields is at
// most 7); X = A ^ B, Y = X + 0x77777777 sets bit 3 of a nibble iff the slot
// mismatches; one PRMT with sign replication turns the two slots' bits into
// 16-bit masks, one LOP3 selects the rebased match / mismatch scores.
//
// Argmax: only the antidiagonal maximum is reduced per step (a VIMNMX3.S16x2
// tree); when it raises best, the killed antidiagonal is copied (predicated
// moves) and the cell (smallest slot holding the maximum, c-amb-9) is decoded
// once, when the task finishes or is handed over.
#pragma once

#include "xdrop_window.cuh"

namespace logan {

constexpr int32_t DEAD16 = -16384;
constexpr uint32_t DEAD2 = 0xC000C000u;
constexpr int32_t PACK_XMAX = 16000;  // live u <= X + 381 < 2^15

// PRMT with the sign-replicate selectors (CUDA's __byte_perm ignores bit 3 of a selector)
__device__ __forceinline__ uint32_t prmt_s(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}

// v's low half in both halves (one PRMT)
#ifdef LOGAN_PK2_MUL
__device__ __forceinline__ uint32_t pk2(int32_t v) { return ((uint32_t)v & 0xffffu) * 0x10001u; }
#else
__device__ __forceinline__ uint32_t pk2(int32_t v) { return __byte_perm((uint32_t)v, 0u, 0x1010u); }
#endif
__device__ __forceinline__ uint32_t vadd2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("add.s16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ int32_t lo16(uint32_t w) { return (int32_t)(int16_t)(w & 0xffffu); }
__device__ __forceinline__ int32_t hi16(uint32_t w) { return ((int32_t)w) >> 16; }

// M2: match - mismatch = 2 (the paper's +1/-1 scoring): the substitution is
// diag + (match - dl) + 2 * mask (two FMA-pipe adds of the sign-replicated
// mismatch mask) instead of a LOP3 select (ALU pipe, the bound)
template <int G, int R, int FMT, bool M2>
struct Window16 {
    static_assert(FMT == LOGAN_SEQ_2BIT, "packed window: 2-bit pools");
    // R = 4 and 8 only as one-warp latency shapes (W = 128, 256): one base word per lane
    static_assert(R % 4 == 0 && R >= 4 && R <= 32 && (R >= 16 || G == 32) && (G & (G - 1)) == 0 && G * R <= 1024,
                  "packed window shape");
    static constexpr int GG = G, W = G * R, H = R / 2;
    static constexpr int CB = 4, FPW = 8;
    static constexpr int NW = (R + FPW - 1) / FPW;
    static constexpr int RL = R - (NW - 1) * FPW;
    static constexpr uint32_t FM = 15u;
    static constexpr uint32_t SA = 4u, SB = 5u;  // 3-bit sentinels: every XOR <= 7

    uint32_t E[H], O[H], C[H];  // even / odd antidiagonal; C: copy of the raising antidiagonal
    uint32_t Aw[NW], Bw[NW];
    WinState<FMT> st;
    int32_t tv, cd, cS0;        // pending argmax: value, antidiagonal (< 0: none), window base
    int gl;
    unsigned gmask;
    const int8_t *tab;          // unused (interface of Window)
    static constexpr int SB_STRIDE = 2 * R + 1;
    int32_t *sbase;

    // slot s of a packed array
    __device__ __forceinline__ static int32_t get(const uint32_t (&a)[H], int s) {
        return s < H ? lo16(a[s]) : hi16(a[s - H]);
    }

    // ---- base fields (as Window, 4-bit, slot order) ---------------------------
    __device__ __forceinline__ static uint32_t top_field(const uint32_t (&w)[NW]) {
        return (w[NW - 1] >> (CB * (RL - 1))) & FM;
    }
    __device__ __forceinline__ static void shift_down(uint32_t (&w)[NW], uint32_t in) {
#pragma unroll
        for (int q = 0; q < NW - 1; ++q) w[q] = __funnelshift_r(w[q], w[q + 1], CB);
        if (RL == FPW) w[NW - 1] = __funnelshift_r(w[NW - 1], in, CB);
        else w[NW - 1] = (w[NW - 1] >> CB) | (in << (CB * (RL - 1)));
    }
    __device__ __forceinline__ static void shift_up(uint32_t (&w)[NW], uint32_t in) {
#pragma unroll
        for (int q = NW - 1; q > 0; --q) w[q] = __funnelshift_l(w[q - 1], w[q], CB);
        w[0] = (w[0] << CB) | in;
        if (RL < FPW) w[NW - 1] &= (1u << (CB * (RL < FPW ? RL : 0))) - 1u;
    }
    __device__ __forceinline__ void load_bases(const Params &P) {
        const int32_t s0 = st.S0 + gl * R;
        const int32_t ch = ceil_half(st.d), fh = floor_half(st.d);
#pragma unroll
        for (int q = 0; q < NW; ++q) { Aw[q] = 0; Bw[q] = 0; }
        st.sa.seek(P, s0 + ch);
#pragma unroll 1
        for (int r = 0; r < R; ++r) shift_down(Aw, st.sa.next(P, SA));
        st.sb.seek(P, fh - (s0 + R - 1));
#pragma unroll 1
        for (int r = R - 1; r >= 0; --r) shift_up(Bw, st.sb.next(P, SB));
        if (gl == G - 1) st.sa.seek(P, st.S0 + W + ch);  // sa.idx = S0 + W + ceil(d/2)
        if (gl == 0) st.sb.seek(P, fh - st.S0 + 1);      // sb.idx = floor(d/2) - S0 + 1
    }

    // ---- task start / hand-over (canonical records, int32 per slot) -----------
    __device__ __forceinline__ void init(const Params &P, uint32_t task) {
        const TaskDesc td = task_desc(P, task);
        st.task = task;
        st.m = td.a.len;
        st.n = td.b.len;
        st.d = 0;
        st.S0 = -(W / 2);
        st.best = 0;
        st.arg_i = st.arg_j = 0;
        st.Tq[0] = st.Tq[1] = -P.xdrop;
        st.K[0] = st.K[1] = KNONE;
        st.KZ[0] = st.KZ[1] = KNONE;
        st.dc[0] = st.dc[1] = 0;
        st.sF[0] = st.sF[1] = EMPTY_F;
        st.sL[0] = st.sL[1] = EMPTY_L;
        st.cells = 0;
        st.shifts = 0;
        st.cells_entry = 0;
        cd = -1;
        // the origin is window slot W/2: lane (W/2) / R, local slot (W/2) % R
        constexpr int OL = (W / 2) / R, OS = (W / 2) % R;
#pragma unroll
        for (int k = 0; k < H; ++k) {
            const bool here = gl == OL && k == OS % H;
            const uint32_t xo = OS < H ? ((uint32_t)(DEAD16 & 0xffff) << 16) | ((uint32_t)P.xdrop & 0xffffu)
                                       : ((uint32_t)P.xdrop << 16) | (uint32_t)(DEAD16 & 0xffff);
            E[k] = here ? xo : DEAD2;
            O[k] = DEAD2;
        }
        st.sa.s = td.a;
        st.sb.s = td.b;
        load_bases(P);
    }

    // the argmax of the last raise (smallest slot of the copied antidiagonal
    // holding the maximum): once per task, at its end or hand-over
    __device__ __forceinline__ void finalize() {
        if (cd < 0) return;
        int s = INT32_MAX;  // the maximum is in the copy: the smallest slot holding it
#pragma unroll
        for (int q = R - 1; q >= 0; --q)
            if (get(C, q) == tv) s = gl * R + q;
        if (G > 1) s = grp_min<G>(s, gmask);
        st.arg_i = cS0 + s + ceil_half(cd);
        st.arg_j = cd - st.arg_i;
        cd = -1;
    }

    __device__ __forceinline__ void save(const Params &P, int32_t *rec) {
        finalize();
        const int32_t d = st.d;
        const int p = d & 1;
#pragma unroll
        for (int s = 0; s < R; ++s) {  // (unrolled: a run-time index would put the arrays in local memory)
            rec[REC_HDR + gl * R + s] = get(E, s);
            rec[REC_HDR + W + gl * R + s] = get(O, s);
        }
        if (gl != 0) return;
        rec[0] = (int32_t)st.task; rec[1] = d; rec[2] = st.S0; rec[3] = st.best;
        rec[4] = st.arg_i; rec[5] = st.arg_j;
        rec[6] = st.best - P.xdrop;
        rec[7] = p ? st.Tq[1] : st.Tq[0];
        rec[8] = p ? st.Tq[0] : st.Tq[1];
        rec[9] = p ? st.sF[1] : st.sF[0];
        rec[10] = p ? st.sL[1] : st.sL[0];
        rec[11] = p ? st.sF[0] : st.sF[1];
        rec[12] = p ? st.sL[0] : st.sL[1];
        rec[13] = 0;
        rec[14] = (int32_t)st.shifts; rec[15] = W;
        rec[16] = (int32_t)(uint32_t)st.cells; rec[17] = (int32_t)(uint32_t)(st.cells >> 32);
    }

    // (the first level never receives records; kept for the interface)
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
        st.Tq[0] = st.Tq[1] = Td1;
        st.best = Td + P.xdrop;
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
        cd = -1;
        int32_t Fm = min(st.sF[0], st.sF[1]), Lm = max(st.sL[0], st.sL[1]);
        if (Fm > Lm) { Fm = S0src; Lm = S0src + Wsrc - 1; }
        st.S0 = ((Fm + Lm) >> 1) - W / 2;
        // best_d > best_{d-1}: d's maximum is re-issued as pending (value only) and
        // the recorded argmax stays (the raise is re-detected and re-decoded from d)
        const int32_t kd = best_d > st.best ? best_d - Td1 : KNONE;
        st.K[0] = p ? KNONE : kd;
        st.K[1] = p ? kd : KNONE;
        const int32_t rb = Td - Td1;
#pragma unroll
        for (int s = 0; s < R; ++s) {
            const int32_t q = st.S0 + gl * R + s - S0src;
            const bool in = q >= 0 && q < Wsrc;
            int32_t ve = in ? rec[REC_HDR + q] : DEAD;
            int32_t vo = in ? rec[REC_HDR + Wsrc + q] : DEAD;
            ve = p == 0 ? ve + rb : ve;
            vo = p == 1 ? vo + rb : vo;
            ve = max(ve, DEAD16 - 2 * 127);
            vo = max(vo, DEAD16 - 2 * 127);
            put_slot(E, s, ve);
            put_slot(O, s, vo);
        }
        load_bases(P);
    }
    __device__ __forceinline__ static void put_slot(uint32_t (&a)[H], int s, int32_t v) {
        const uint32_t h = (uint32_t)v & 0xffffu;
        if (s < H) a[s] = (a[s] & 0xffff0000u) | h;
        else a[s - H] = (a[s - H] & 0xffffu) | (h << 16);
    }

    // ---- pending maxima ---------------------------------------------------------
    // Fold the pending maximum k (a value relative to T) of raw antidiagonal a,
    // whose killed values (shifted by -dla) are in array `arr`: a raise copies it.
    __device__ __forceinline__ void fold(int32_t k, int32_t T, int32_t a, int32_t dla, const uint32_t (&arr)[H]) {
        const bool raise = k > st.best - T;  // k = KNONE never raises
        if (raise) {
            st.best = k + T;
            tv = k - dla;
            cd = a;
            cS0 = st.S0;
        }
#pragma unroll
        for (int q = 0; q < H; ++q) C[q] = raise ? arr[q] : C[q];
    }

    // Dead-slot mask of a killed array in "pair order": one PRMT takes the sign
    // bytes of word j and word j + H/2 (slots j, j + H/2, j + H, j + 3H/2, each
    // replicated to a whole byte) and one LOP3 keeps bit j of every byte, so bit
    // 8b + j is slot (H/2) b + j. The bit order is monotone in the slot order: the
    // first / last live slot are one FLO away (two ALU instructions per word pair;
    // the earlier nibble layout took four plus a branchy decode).
    static constexpr int HH = H / 2;
    static constexpr uint32_t USED = 0x01010101u * ((1u << HH) - 1u);  // bits that hold a slot
    __device__ __forceinline__ static uint32_t dead_m(const uint32_t (&a)[H]) {
        uint32_t z = 0;
#pragma unroll
        for (int j = 0; j < HH; ++j) {
            const uint32_t g = prmt_s(a[j], a[j + HH], 0xFBD9u);  // sign bytes: j lo, j+HH lo, j hi, j+HH hi
            z |= g & (0x01010101u << j);
        }
        return z;
    }
    __device__ __forceinline__ static int32_t bit_slot(int32_t b) {
        return HH == 8 ? b : HH * (b >> 3) + (b & 7);
    }
    __device__ __forceinline__ static int32_t slot_bit(int32_t s) {
        return HH == 8 ? s : 8 * (s / HH) + s % HH;
    }

    // live extremes of the killed antidiagonal e-1 (parity Qp) in array a:
    // sF / sL[Qp] (validity-masked: cells past the matrix do not count)
    template <int Qp>
    __device__ __forceinline__ void extremes(int32_t e, const uint32_t (&a)[H]) {
        const uint32_t z = dead_m(a);
        const int32_t chq = e >> 1, fhq = (e - 1) >> 1;  // ceil((e-1)/2), floor((e-1)/2)
        const int32_t vlo = fhq - st.n, vhi = st.m - chq;
        const int32_t base = st.S0 + gl * R;
        uint32_t vmask = USED;
        if (vlo > base || vhi < base + R - 1) {  // near the matrix edges: valid slots [rlo, rhi]
            const int32_t rlo = max(vlo - base, 0), rhi = min(vhi - base, R - 1);
            const int32_t blo = slot_bit(rlo), bhi = slot_bit(rhi);
            vmask = (rlo <= rhi) ? ((0xffffffffu >> (31 - bhi)) & ~((1u << blo) - 1u) & USED) : 0u;
        }
        const uint32_t live = ~z & vmask;
        bool h = live != 0;
        int32_t f = bit_slot(__ffs(live) - 1), l = bit_slot(31 - __clz(live));
        if (G > 1) {  // group extremes (sentinels for lanes without a live slot)
            f = grp_min<G>(h ? gl * R + f : INT32_MAX, gmask);
            l = grp_max<G>(h ? gl * R + l : INT32_MIN, gmask);
            h = f != INT32_MAX;
        }
        st.sF[Qp] = h ? st.S0 + f : EMPTY_F;
        st.sL[Qp] = h ? st.S0 + l : EMPTY_L;
    }

    template <int PAR>
    __device__ __forceinline__ int step(const Params &P, bool force) {
        const int32_t e = st.d + 1;
        constexpr int Q = 1 - PAR;

        // (a) best_{e-2} from the pending maximum of raw e-2 (relative to T_{e-3});
        //     the killed e-2 (array of parity PAR) is copied on a raise
        const int32_t T3 = st.Tq[Q], T2 = st.Tq[PAR];
        if (PAR) fold(st.K[PAR], T3, e - 2, T2 - T3, O);
        else fold(st.K[PAR], T3, e - 2, T2 - T3, E);
        st.K[PAR] = KNONE;
        const int32_t T1 = st.best - P.xdrop;
        const int32_t dl = T1 - T2;
        const uint32_t ndl2 = pk2(-dl);

        // (b) late kill of e-1
        if (PAR) {
#pragma unroll
            for (int k = 0; k < H; ++k) E[k] = __viaddmin_u16x2(E[k], ndl2, DEAD2);
        } else {
#pragma unroll
            for (int k = 0; k < H; ++k) O[k] = __viaddmin_u16x2(O[k], ndl2, DEAD2);
        }
        st.Tq[Q] = T1;

        // (c) odd e: the window check of Window::step needs the live extremes of e-1
        //     and e-2 only at the window's edges: slots 0 and R-1 both dead in both
        //     arrays (a sign test) means nothing to do, and the raw cells of e need not
        //     wait for the extremes. Otherwise (numerically live edge slots, which can
        //     also be cells past the matrix) the rare path takes the exact decision.
        if (PAR == 1) {
            // an edge slot counts only inside the matrix on e-1 (slot 0 has the
            // largest j, slot R-1 the largest i); e-2's validity range differs from
            // e-1's by at most one slot on each side, which only makes this test
            // more eager (the exact decision below is unaffected)
            const uint32_t lo0 = E[0] & O[0], hiR = E[H - 1] & O[H - 1];
            const bool in0 = st.S0 >= ((e - 1) >> 1) - st.n, inR = st.S0 + W - 1 <= st.m - (e >> 1);
            bool edge = (gl == 0 && !(lo0 & 0x8000u) && in0) || (gl == G - 1 && !(hiR & 0x80000000u) && inR);
            // (a shuffle, not a ballot: __ballot_sync over a per-group mask compiles to
            //  WARPSYNC.EXCLUSIVE, which serialises the groups of the warp)
            if (G > 1) edge = (__shfl_sync(gmask, int(edge), 0, G) | __shfl_sync(gmask, int(edge), G - 1, G)) != 0;
            if (force || edge) {
                extremes<Q>(e, E);
                if (st.sF[0] == EMPTY_F && st.sF[1] == EMPTY_F) return 1;  // P:186, c-amb-7
                bool ho = force;
                if (!ho) {
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
                if (ho) {
                    fold(st.K[Q], T2, e - 1, dl, E);  // e-1 is even here: array E (killed above)
                    st.K[Q] = KNONE;
                    return 2;
                }
            }
        }

        // (e) bases for antidiagonal e (lane G-1 reads the A stream, lane 0 the B one)
        if (PAR == 1) {
            uint32_t in = 0;
            if (G > 1) in = __shfl_down_sync(gmask, Aw[0], 1, G) & FM;
            const uint32_t x = st.sa.next_fast(SA);
            if (gl == G - 1) in = x;
            shift_down(Aw, in);
        } else {
            uint32_t in = 0;
            if (G > 1) in = __shfl_up_sync(gmask, top_field(Bw), 1, G);
            const uint32_t x = st.sb.next_fast(SB);
            if (gl == 0) in = x;
            shift_up(Bw, in);
        }

        // (f) raw cells of e (relative to T_{e-1}), two slots per instruction
#ifdef LOGAN_OLD_CONST
        const uint32_t gap2 = pk2(P.gap);
        const uint32_t fg2 = pk2(DEAD16 - P.gap);
        const uint32_t sma2 = pk2(P.match - dl), smi2 = pk2(P.mismatch - dl);
#else
        const uint32_t gap2 = P.gap2;
        const uint32_t fg2 = P.fg2;
        // (match - dl, mismatch - dl in both halves: two FMA-pipe adds of the packed constants)
        const uint32_t sma2 = vadd2(P.match2, ndl2), smi2 = vadd2(P.mis2, ndl2);
#endif
        // (FMA-pipe IMADs with an opaque run-time 1 / 16: the ALU pipe is the bound)
        const uint32_t one = (uint32_t)P.one, sixteen = (uint32_t)P.one << 4;
        uint32_t Y[NW], Yl[NW];
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            // bit 3 of a nibble: the slot mismatches
            asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(Y[q]) : "r"(Aw[q] ^ Bw[q]), "r"(one), "r"(0x77777777u));
            asm("mad.lo.u32 %0, %1, %2, 0;" : "=r"(Yl[q]) : "r"(Y[q]), "r"(sixteen));
        }
        // the seam words' neighbours from the adjacent lanes (DEAD beyond the window)
        uint32_t nbr = DEAD2;
        if (G > 1) {
            if (PAR == 1) { nbr = __shfl_down_sync(gmask, E[0], 1, G); if (gl == G - 1) nbr = DEAD2; }
            else { nbr = __shfl_up_sync(gmask, O[H - 1], 1, G); if (gl == 0) nbr = DEAD2; }
        }
#pragma unroll
        for (int k = 0; k < H; ++k) {
            // mismatch masks of slots k (low half) and k + H (high half)
            const int s0 = k, s1 = k + H;
            const uint32_t a = (s0 & 1) ? Y[s0 / 8] : Yl[s0 / 8];
            const uint32_t b = (s1 & 1) ? Y[s1 / 8] : Yl[s1 / 8];
            const uint32_t b0 = (uint32_t)((s0 % 8) >> 1), b1 = (uint32_t)((s1 % 8) >> 1);
            const uint32_t sel = (8u | b0) | ((8u | b0) << 4) | ((12u | b1) << 8) | ((12u | b1) << 12);
            const uint32_t mask2 = prmt_s(a, b, sel);
            uint32_t s2;
            if (M2) s2 = vadd2(mask2, mask2);  // -2 or 0 per half; sma2 added below
            else asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(s2) : "r"(mask2), "r"(smi2), "r"(sma2));
            uint32_t up, left, diag;
            if (PAR == 1) {  // odd e: up = E[s+1], left = E[s], diag = O[s]
                // seam: (slot H of this lane, slot 0 of the next lane)
                up = (k < H - 1) ? E[k + 1] : __byte_perm(E[0], nbr, 0x5432);
                left = E[k];
                diag = O[k];
            } else {         // even e: up = O[s], left = O[s-1], diag = E[s]
                up = O[k];
                // seam: (slot R-1 of the previous lane, slot H-1 of this lane)
                left = (k > 0) ? O[k - 1] : __byte_perm(nbr, O[H - 1], 0x5432);
                diag = E[k];
            }
            const uint32_t t0 = __vimax3_s16x2(up, left, fg2);
            uint32_t dps;
            asm("add.s16x2 %0, %1, %2;" : "=r"(dps) : "r"(diag), "r"(s2));
            if (M2) dps = vadd2(dps, sma2);
            const uint32_t u = __viaddmax_s16x2(t0, gap2, dps);
            if (PAR == 1) O[k] = u;
            else E[k] = u;
        }
        // note: the even step reads O[k-1] after O[k] ... O is not written in an
        // even step (it writes E), and the odd step reads E only (writes O): safe

        // (g) the maximum of raw e, pending until step e + 2
        uint32_t mx[(H + 2) / 3];
#pragma unroll
        for (int q = 0; q < (H + 2) / 3; ++q) {
            const uint32_t x0 = PAR ? O[3 * q] : E[3 * q];
            const uint32_t x1 = (3 * q + 1 < H) ? (PAR ? O[3 * q + 1] : E[3 * q + 1]) : x0;
            const uint32_t x2 = (3 * q + 2 < H) ? (PAR ? O[3 * q + 2] : E[3 * q + 2]) : x0;
            mx[q] = __vimax3_s16x2(x0, x1, x2);
        }
        constexpr int NM = (H + 2) / 3;
        uint32_t m2 = mx[0];
#pragma unroll
        for (int q = 1; q < NM; q += 2)
            m2 = __vimax3_s16x2(m2, mx[q], (q + 1 < NM) ? mx[q + 1] : mx[q]);
        int32_t kmx = max(lo16(m2), hi16(m2));
        if (G > 1) kmx = grp_max<G>(kmx, gmask);
        st.K[PAR] = kmx;

        // (b') live extremes of e-1 (band bookkeeping, off the cells' critical path)
        if (PAR) extremes<Q>(e, E);
        else extremes<Q>(e, O);
        // termination after an even e-1 (c-amb-7): e-1 and e-2 both empty;
        // best_{e-2} is final and the raw cells of e just computed are discarded
        if (PAR == 1 && st.sF[0] == EMPTY_F && st.sF[1] == EMPTY_F) return 1;

        // (d) band cells of e (c-amb-14)
        {
            const int32_t c = PAR ? (e - 1) >> 1 : e >> 1;
            const int32_t F1 = st.sF[Q], F2 = st.sF[PAR], L1 = st.sL[Q], L2 = st.sL[PAR];
            const int32_t fmin = PAR ? min(F1, F2 + 1) : min(F1, F2);
            const int32_t lmax = PAR ? max(L1, L2) : max(L1, L2 - 1);
            const int32_t lo = __vimax3_s32(fmin + c, 1, e - st.n);
            const int32_t hi = __vimin3_s32(lmax + c + 1, st.m, e - 1);
            st.cells += (uint32_t)__vimax_s32_relu(hi - lo + 1, 0);
        }

        st.d = e;
        return 0;
    }

    // ---- window shifts (rare): in the split layout a shift by one slot moves
    // whole words (both halves together), plus one PRMT at the seam. The words go
    // through this thread's shared-memory slice so that the reloads land in the
    // registers the arrays already occupy (a register rotation here makes the
    // compiler copy both arrays on every step's common path)
    __device__ __forceinline__ void shift_slots(int by) {
        uint32_t ne = DEAD2, no = DEAD2;  // the adjacent lane's word entering at the seam
        if (G > 1) {
            if (by > 0) {
                ne = __shfl_down_sync(gmask, E[0], 1, G);
                no = __shfl_down_sync(gmask, O[0], 1, G);
                if (gl == G - 1) ne = no = DEAD2;
            } else {
                ne = __shfl_up_sync(gmask, E[H - 1], 1, G);
                no = __shfl_up_sync(gmask, O[H - 1], 1, G);
                if (gl == 0) ne = no = DEAD2;
            }
        }
        volatile uint32_t *b = (volatile uint32_t *)sbase;
#pragma unroll
        for (int k = 0; k < H; ++k) { b[k] = E[k]; b[H + k] = O[k]; }
        if (by > 0) {  // new slot s = old slot s + 1
#pragma unroll
            for (int k = 0; k < H - 1; ++k) { E[k] = b[k + 1]; O[k] = b[H + k + 1]; }
            E[H - 1] = __byte_perm(b[0], ne, 0x5432);  // (old slot H, the next lane's old slot 0)
            O[H - 1] = __byte_perm(b[H], no, 0x5432);
        } else {       // new slot s = old slot s - 1
#pragma unroll
            for (int k = 1; k < H; ++k) { E[k] = b[k - 1]; O[k] = b[H + k - 1]; }
            E[0] = __byte_perm(ne, b[H - 1], 0x5432);  // (the previous lane's old slot R-1, old slot H-1)
            O[0] = __byte_perm(no, b[2 * H - 1], 0x5432);
        }
    }
    __device__ __forceinline__ void shift_right(const Params &P, int32_t d) {
        uint32_t aIn = 0, bIn = 0;
        if (G > 1) {
            aIn = __shfl_down_sync(gmask, Aw[0], 1, G) & FM;
            bIn = __shfl_down_sync(gmask, Bw[0], 1, G) & FM;
        }
        const int32_t S1 = st.S0 + 1;
        if (gl == G - 1) {
            aIn = st.sa.next(P, SA);  // a_{S1 + W - 1 + ceil(d/2)}
            bIn = seq_at<FMT>(P, st.sb.s, floor_half(d) - S1 - (W - 1), SB);
        }
        if (gl == 0) st.sb.seek(P, st.sb.idx - 1);  // b stream steps back one base
        shift_slots(+1);
        shift_down(Aw, aIn);
        shift_down(Bw, bIn);
        st.S0 = S1;
        ++st.shifts;
    }
    __device__ __forceinline__ void shift_left(const Params &P, int32_t d) {
        uint32_t aIn = 0, bIn = 0;
        if (G > 1) {
            aIn = __shfl_up_sync(gmask, top_field(Aw), 1, G);
            bIn = __shfl_up_sync(gmask, top_field(Bw), 1, G);
        }
        const int32_t S1 = st.S0 - 1;
        if (gl == 0) {
            aIn = seq_at<FMT>(P, st.sa.s, S1 + ceil_half(d), SA);
            bIn = st.sb.next(P, SB);  // b_{floor(d/2) - S1}
        }
        if (gl == G - 1) st.sa.seek(P, st.sa.idx - 1);  // a stream steps back one base
        shift_slots(-1);
        shift_up(Aw, aIn);
        shift_up(Bw, bIn);
        st.S0 = S1;
        ++st.shifts;
    }
};

}  // namespace logan
