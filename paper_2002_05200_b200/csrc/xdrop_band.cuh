// xdrop_band.cuh — level 7, wide bands: one CTA per task sweeps the band as
// packed int16 pairs held in a shared-memory ring (stage 1: one warp per task,
// 4096 slots; stage 2, for the bands that outgrow it: four warps, 8192 slots).
//
// Same method and cell rule as the register windows (eq. P:85, drop rule P:89,
// best after the complete antidiagonal P:178, band trimming and termination
// P:186, c-amb-6/7), the same threshold-relative values u = S - T_d and the
// same diagonal-slot coordinates (slot s on antidiagonal d is i = s + ceil(d/2),
// j = floor(d/2) - s; see xdrop_window.cuh). This level is for bands too wide
// for registers: the paper's X = 500 ... 5000 sweep (SURVEY §8f
// row 1), where the band is the whole antidiagonal of the extension's matrix.
//
// B200 design:
//  * Values are int16 in a ring of SLOTS slots per parity (BandCfg); slot s
//    lives at ring index s mod SLOTS, two slots per 32-bit word, so the band
//    never has to be re-centred. Live u <= X + 2*127 < 2^15 for X <= 30000;
//    every dead value is exactly D16 = -16384.
//  * The cell runs on the pairs directly (DPX .S16x2: VIMNMX3, VIADDMNMX, and
//    VIMNMX.U16x2 for the exact kill): two cells per instruction and no
//    unpack / pack. The floor max(up, left, D16 - gap') keeps every
//    intermediate inside int16 (|gap'|, |s'| <= 381), so nothing wraps.
//  * Bases are staged per task in two circular shared-memory buffers, one code
//    per nibble (2-bit pool) or byte (u8 pool): a_i at position i, b_j at
//    position -j, so the 8 codes of a lane's 8 slots are one funnel shift of
//    two words for either read. A mismatch mask per slot pair comes from
//    (A ^ B) + 0x77777777 and one PRMT with sign replication; the substitution
//    score pair is a LOP3 select between the rebased match / mismatch pairs.
//  * Per antidiagonal the CTA visits only the slots that can be live (the
//    predecessors' live extents widened by one, clipped to the matrix) and
//    clears the ones written two antidiagonals ago that fell outside; thread t
//    takes the 8-slot chunk base + 8t of every 8*NT-slot pass. Per chunk it
//    keeps a packed (max, first chunk) key and the first / last live chunk;
//    warp CREDUX, one __syncthreads on parity-double-buffered partials, and
//    every thread folds the NW partials: best, the threshold and the
//    chunk-granular live extents (which bound the next visited range) are
//    uniform without a second barrier.
//  * Warp 0 alone turns the chunk extents into exact live extents (one
//    broadcast LDS.128 per chunk and a sign PRMT) for the cell count
//    (c-amb-14), and finds the exact argmax slot when best rises.
//  * A band wider than the ring (minus a margin), or X > BAND_XMAX, goes to
//    the CTA level (restart).
#pragma once

#include "xdrop_common.cuh"
#include "xdrop_window.cuh"

namespace logan {

constexpr int BAND_XMAX = 30000;              // live u <= X + 2*127 must fit int16
constexpr int BAND_MARGIN = 128;              // slots kept free between the band's ends
#ifndef LOGAN_BAND_PAD
#define LOGAN_BAND_PAD 48
#endif
constexpr int BAND_PAD = LOGAN_BAND_PAD;      // codes staged beyond the needed range
constexpr uint32_t D16X2 = 0xC000C000u;       // two dead slots (-16384 each)

// Launch configuration of the band level: threads per task (= per block) and
// ring slots per parity. The band level runs in two stages (logan_impl.cuh):
// one warp per task with a 4096-slot ring (20 KB of shared memory: 11 tasks per
// SM; no barrier waits, the per-antidiagonal scalar work done once per task
// instead of once per warp), then the bands that outgrow it on 4 warps with an
// 8192-slot ring. Code positions per read buffer (circular): the codes a planned
// antidiagonal needs span at most SLOTS - BAND_MARGIN + 2 positions; with
// BAND_PAD of slack on both sides and word rounding they must fit CAP.
template <int NT_, int SLOTS_>
struct BandCfg {
    static constexpr int NT = NT_, NW = NT_ / 32;
    static constexpr int ARG_WARP = NW > 1 ? 1 : 0;  // the warp that keeps the argmax
    static constexpr int SLOTS = SLOTS_, WORDS = SLOTS_ / 2, CAP = SLOTS_;
    static_assert(SLOTS - BAND_MARGIN + 2 + 2 * BAND_PAD + 16 <= CAP, "code buffer too small for the ring");
};
using BandSmall = BandCfg<32, 4096>;
using BandBig = BandCfg<128, 8192>;

template <int FMT> struct BandFmt;
template <> struct BandFmt<LOGAN_SEQ_2BIT> { static constexpr int CB = 4; };  // one nibble per base
template <> struct BandFmt<LOGAN_SEQ_U8> { static constexpr int CB = 8; };    // one byte per base

// Shared-memory layout (32-bit words). Each code buffer has CAPW words plus
// MIRROR copies of its first words behind the end, so the words a chunk needs
// are consecutive without a second wrap.
template <int FMT, class C>
struct BandSmem {
    static constexpr int CB = BandFmt<FMT>::CB;
    static constexpr int CPW = 32 / CB;                 // codes per word
    static constexpr int CAPW = C::CAP / CPW;         // words per read buffer
    static constexpr int MIRROR = 4;
    static constexpr size_t VAL = 0;                    // uint32 val[2][C::WORDS]
    static constexpr size_t CA = VAL + 2 * C::WORDS;  // uint32 ca[CAPW + MIRROR]
    static constexpr size_t CBUF = CA + CAPW + MIRROR;  // uint32 cb[CAPW + MIRROR]
    static constexpr size_t RED = CBUF + CAPW + MIRROR; // int4 red[2][C::NW]
    static constexpr size_t WORDS = RED + 2 * C::NW * 4;
    static constexpr size_t BYTES = WORDS * sizeof(uint32_t);
    static_assert(RED % 4 == 0, "int4 alignment");
};

extern __shared__ uint4 band_smem[];

// ---- int16x2 helpers (DPX on sm_100a) ---------------------------------------
__device__ __forceinline__ uint32_t pair16(int32_t v) { return ((uint32_t)v & 0xffffu) * 0x10001u; }
__device__ __forceinline__ uint32_t vmax16(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.s16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t vminu16(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
// PRMT in its default mode: selector nibble bit 3 replicates the byte's sign
// (__byte_perm masks that bit off)
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
__device__ __forceinline__ int32_t sext_lo(uint32_t w) { return (int32_t)(int16_t)(w & 0xffffu); }
__device__ __forceinline__ int32_t sext_hi(uint32_t w) { return (int32_t)w >> 16; }

// Mismatch masks of the 4 slot pairs of a chunk: mk[k] has 0xffff in the half
// of slot 2k (low) / 2k+1 (high) iff the two codes differ.
template <int FMT, class C> struct BandCodes;

template <class C> struct BandCodes<LOGAN_SEQ_2BIT, C> {
    using S = BandSmem<LOGAN_SEQ_2BIT, C>;
    uint32_t x;  // nibble r = code of slot s0 + r
    // the chunk's codes start at position q = 8 * c8 + off: word c8 + (off >> 3),
    // bit offset 4 * (off & 7)
    __device__ __forceinline__ static int32_t wstep() { return 1; }
    __device__ __forceinline__ void load(const uint32_t *buf, int32_t w, uint32_t sh) {
        const uint32_t *p = buf + (w & (S::CAPW - 1));
        x = __funnelshift_r(p[0], p[1], sh);
    }
    __device__ __forceinline__ static int32_t word_off(int32_t off) { return off >> 3; }
    __device__ __forceinline__ static uint32_t bit_off(int32_t off) { return 4u * (uint32_t)(off & 7); }
    __device__ __forceinline__ static void masks(const BandCodes &a, const BandCodes &b, uint32_t (&mk)[4]) {
        // codes are 0..3: ((a ^ b) & 3) + 7 per nibble sets the nibble's bit 3 iff
        // they differ and never carries. The & 3 (one LOP3 with the XOR) matters:
        // nibbles of slots outside the staged code range hold stale shared memory,
        // and a stale nibble > 8 would carry into the flag of the slot above it
        // (those slots are masked dead afterwards, their neighbours are not).
        // z has slot 2k+1's flag at bit 7 of byte k, z << 4 has slot 2k's flag there
        const uint32_t z = ((a.x ^ b.x) & 0x33333333u) + 0x77777777u;
        const uint32_t z4 = z << 4;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            mk[k] = prmt(z4, z, (8u + k) | ((8u + k) << 4) | ((12u + k) << 8) | ((12u + k) << 12));
    }
};

template <class C> struct BandCodes<LOGAN_SEQ_U8, C> {
    using S = BandSmem<LOGAN_SEQ_U8, C>;
    uint32_t lo, hi;  // byte r = code of slot s0 + r
    // the chunk's codes start at position q = 8 * c8 + off: word 2 * c8 + (off >> 2)
    __device__ __forceinline__ static int32_t wstep() { return 2; }
    __device__ __forceinline__ void load(const uint32_t *buf, int32_t w, uint32_t sh) {
        const uint32_t *p = buf + (w & (S::CAPW - 1));
        lo = __funnelshift_r(p[0], p[1], sh);
        hi = __funnelshift_r(p[1], p[2], sh);
    }
    __device__ __forceinline__ static int32_t word_off(int32_t off) { return off >> 2; }
    __device__ __forceinline__ static uint32_t bit_off(int32_t off) { return 8u * (uint32_t)(off & 3); }
    __device__ __forceinline__ static uint32_t nonzero_bytes(uint32_t x) {  // bit 7 of byte = (byte != 0)
        return ((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x;
    }
    __device__ __forceinline__ static void masks(const BandCodes &a, const BandCodes &b, uint32_t (&mk)[4]) {
        const uint32_t z0 = nonzero_bytes(a.lo ^ b.lo), z1 = nonzero_bytes(a.hi ^ b.hi);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            mk[k] = prmt(z0, z1, (8u + 2 * k) | ((8u + 2 * k) << 4) | ((9u + 2 * k) << 8) | ((9u + 2 * k) << 12));
    }
};

// Per-task state, uniform over the CTA (warp-0-only fields marked).
struct BandTask {
    uint32_t task;
    SeqRef a, b;
    int32_t m, n, d;
    int32_t best;
    int32_t Tn, Tq[2];         // as in WinState
    int32_t cF[2], cL[2];      // chunk-granular live extents of the last antidiagonal of each parity
    int32_t Dlo[2], Dhi[2];    // slots written (possibly non-dead) in each parity's array
    int32_t fa_lo, fa_hi;      // staged code ranges (unwrapped positions)
    int32_t fb_lo, fb_hi;
    // warp 0 only: exact live extents, argmax, cell count
    int32_t xF[2], xL[2];
    int32_t arg_i, arg_j;
    uint64_t cells, cells_entry;
};

template <int FMT, class C>
struct BandCta {
    using S = BandSmem<FMT, C>;
    using Codes = BandCodes<FMT, C>;
    int tid, lane, warp;
    BandTask t;

    __device__ __forceinline__ static uint32_t *sm() { return (uint32_t *)band_smem; }
    __device__ __forceinline__ static uint32_t *val(int p) { return sm() + S::VAL + p * C::WORDS; }
    __device__ __forceinline__ static uint32_t *ca() { return sm() + S::CA; }
    __device__ __forceinline__ static uint32_t *cb() { return sm() + S::CBUF; }
    __device__ __forceinline__ static int4 *red(int p) { return (int4 *)(sm() + S::RED) + p * C::NW; }

    // Stage the codes of unwrapped positions [q_lo, q_hi) into buf: a uses
    // code(q) = a_q, b uses code(q) = b_{-q}; positions outside the read hold 0
    // (only cells inside the matrix ever use a code).
    __device__ __forceinline__ void stage(const Params &P, uint32_t *buf, const SeqRef &s, int sign,
                                          int32_t q_lo, int32_t q_hi) const {
        constexpr int CPW = S::CPW, CB = S::CB;
        const int32_t w0 = q_lo >> (CB == 4 ? 3 : 2), w1 = (q_hi - 1) >> (CB == 4 ? 3 : 2);
#pragma unroll 1
        for (int32_t w = w0 + tid; w <= w1; w += C::NT) {
            uint32_t x = 0;
#pragma unroll 1
            for (int r = 0; r < CPW; ++r) {
                const int32_t q = w * CPW + r;
                x |= seq_at<FMT>(P, s, sign > 0 ? q : -q, 0u) << (CB * r);
            }
            const int32_t wi = w & (S::CAPW - 1);
            buf[wi] = x;
            if (wi < S::MIRROR) buf[S::CAPW + wi] = x;
        }
    }

    __device__ __forceinline__ void begin(const Params &P, uint32_t task) {
        const TaskDesc td = task_desc(P, task);
        t.task = task;
        t.a = td.a;
        t.b = td.b;
        t.m = td.a.len;
        t.n = td.b.len;
        t.fa_lo = t.fa_hi = t.fb_lo = t.fb_hi = 0;  // nothing staged
        uint4 *v4 = (uint4 *)val(0);
        const uint4 z = make_uint4(D16X2, D16X2, D16X2, D16X2);
#pragma unroll 4
        for (int q = tid; q < 2 * C::WORDS / 4; q += C::NT) v4[q] = z;
        if (P.poison) {  // test knob: code buffers start as garbage (stale smem is arbitrary)
            for (int q = tid; q < 2 * (S::CAPW + S::MIRROR); q += C::NT) ca()[q] = 0xffffffffu;  // every nibble 15: the worst case for the mismatch-flag carry
        }
        __syncthreads();
    }

    // fresh start at antidiagonal 0: the origin S(0,0) = 0, u = 0 - T_0 = X
    __device__ __forceinline__ void init(const Params &P, uint32_t task) {
        begin(P, task);
        t.d = 0;
        t.best = 0;
        t.arg_i = t.arg_j = 0;
        t.Tq[0] = t.Tq[1] = t.Tn = -P.xdrop;
        t.cF[0] = t.cL[0] = t.xF[0] = t.xL[0] = 0;
        t.cF[1] = t.xF[1] = EMPTY_F;
        t.cL[1] = t.xL[1] = EMPTY_L;
        t.Dlo[0] = t.Dhi[0] = 0;
        t.Dlo[1] = EMPTY_F;
        t.Dhi[1] = EMPTY_L;
        t.cells = t.cells_entry = 0;
        if (tid == 0) val(0)[0] = (D16X2 & 0xffff0000u) | ((uint32_t)P.xdrop & 0xffffu);
        __syncthreads();
    }

    // continue a task handed over by a register window (record: xdrop_window.cuh)
    __device__ __forceinline__ void resume(const Params &P, const int32_t *rec) {
        begin(P, (uint32_t)rec[0]);
        t.d = rec[1];
        const int32_t S0src = rec[2];
        t.best = rec[3];
        t.arg_i = rec[4];
        t.arg_j = rec[5];
        const bool odd = t.d & 1;
        t.Tn = rec[6];
        t.Tq[0] = odd ? rec[8] : rec[7];
        t.Tq[1] = odd ? rec[7] : rec[8];
        t.xF[0] = t.cF[0] = odd ? rec[11] : rec[9];
        t.xF[1] = t.cF[1] = odd ? rec[9] : rec[11];
        t.xL[0] = t.cL[0] = odd ? rec[12] : rec[10];
        t.xL[1] = t.cL[1] = odd ? rec[10] : rec[12];
        const int32_t Wsrc = rec[15];
        t.cells = (uint64_t)(uint32_t)rec[16] | ((uint64_t)(uint32_t)rec[17] << 32);
        t.cells_entry = t.cells;
        uint16_t *v0 = (uint16_t *)val(0), *v1 = (uint16_t *)val(1);
        for (int q = tid; q < Wsrc; q += C::NT) {
            const int32_t ri = (S0src + q) & (C::SLOTS - 1);
            // live values are < 2^15 (X <= BAND_XMAX); every dead value becomes D16
            const int32_t e = rec[REC_HDR + q], o = rec[REC_HDR + Wsrc + q];
            v0[ri] = (uint16_t)(e < 0 ? -16384 : e);
            v1[ri] = (uint16_t)(o < 0 ? -16384 : o);
        }
        t.Dlo[0] = t.Dlo[1] = S0src;
        t.Dhi[0] = t.Dhi[1] = S0src + Wsrc - 1;
        __syncthreads();
    }

    // First / last live slot of the chunk at slot c (8-aligned) of array p:
    // sign-replicated high bytes of the four pairs give one dead flag per slot.
    __device__ __forceinline__ void chunk_live(int p, int32_t c, uint32_t &live0, uint32_t &live1) const {
        const uint4 w = *(const uint4 *)(val(p) + ((c >> 1) & (C::WORDS - 1)));
        live0 = ~prmt(w.x, w.y, 0xFDB9u);  // bytes: slots 0..3, 0xff = live
        live1 = ~prmt(w.z, w.w, 0xFDB9u);  // slots 4..7
    }

    // One antidiagonal d = t.d + 1 of parity PAR. Returns 0 = continue,
    // 1 = finished, 2 = band too wide for the ring.
    template <int PAR>
    __device__ __forceinline__ int step(const Params &P) {
        const int32_t d = t.d + 1;
        const int32_t ch = PAR ? (d + 1) >> 1 : d >> 1, fh = PAR ? (d - 1) >> 1 : d >> 1;

        // (1) band cells of d from the exact live extents of d-1, d-2 (warp 0:
        //     the only warp that holds them; c-amb-14, as in the register windows)
        if (warp == 0) {
            const int32_t c1 = PAR ? (d - 1) >> 1 : d >> 1;
            const int32_t c2 = PAR ? (d - 1) >> 1 : (d - 2) >> 1;
            const int32_t lo = max(min(t.xF[1 - PAR] + c1, t.xF[PAR] + c2 + 1), max(1, d - t.n));
            const int32_t hi = min(max(t.xL[1 - PAR] + c1, t.xL[PAR] + c2) + 1, min(t.m, d - 1));
            t.cells += (uint32_t)max(hi - lo + 1, 0);
        }

        // (2) slots that can be live (a live predecessor at d-1 -- even d reads
        //     slots s-1 and s, odd d reads s and s+1 -- or at d-2, slot s), from
        //     the chunk-granular extents (a superset), clipped to the matrix
        const int32_t F1 = t.cF[1 - PAR], L1 = t.cL[1 - PAR], F2 = t.cF[PAR], L2 = t.cL[PAR];
        int32_t vlo = PAR ? min(F1 - 1, F2) : min(F1, F2);
        int32_t vhi = PAR ? max(L1, L2) : max(L1 + 1, L2);
        vlo = max(vlo, max(-ch, fh - t.n));
        vhi = min(vhi, min(t.m - ch, fh));
        int32_t hlo = t.Dlo[PAR], hhi = t.Dhi[PAR];  // and last time's slots (cleared)
        if (vlo <= vhi) { hlo = min(hlo, vlo); hhi = max(hhi, vhi); }

        // (3) codes for the visited cells: a_i, i in [vlo + ch, vhi + ch];
        //     b_j, -j in [vlo - fh, vhi - fh] (uniform check, rare refill)
        if (vlo <= vhi) {
            const int32_t alo = vlo + ch, ahi = vhi + ch + 1, blo = vlo - fh, bhi = vhi - fh + 1;
            const bool ra = alo < t.fa_lo || ahi > t.fa_hi, rb = blo < t.fb_lo || bhi > t.fb_hi;
            if (ra || rb) {
                if (ra) {
                    t.fa_lo = alo - BAND_PAD;
                    t.fa_hi = ahi + BAND_PAD;
                    stage(P, ca(), t.a, +1, t.fa_lo, t.fa_hi);
                }
                if (rb) {
                    t.fb_lo = blo - BAND_PAD;
                    t.fb_hi = bhi + BAND_PAD;
                    stage(P, cb(), t.b, -1, t.fb_lo, t.fb_hi);
                }
                __syncthreads();
            }
        }

        // (4) rebased constants (xdrop_window.cuh step (3)), as int16 pairs
        const int32_t Tc = t.Tn;
        const int32_t gp = P.gap - (Tc - t.Tq[1 - PAR]);
        const int32_t sma = P.match - (Tc - t.Tq[PAR]);
        const int32_t smi = P.mismatch - (Tc - t.Tq[PAR]);
        const uint32_t gp2 = pair16(gp), sma2 = pair16(sma), smi2 = pair16(smi);
        const uint32_t fg2 = pair16(-16384 - gp);  // max(up, left, fg) + gp >= D16: the floor

        uint32_t *cur = val(PAR);               // d-2 in, d out (in place)
        const uint32_t *oth = val(1 - PAR);     // d-1
        const int32_t hbase = hlo & ~7;
        const int32_t c8base = hbase >> 3, c8last = hhi >> 3;  // chunk = 8 slots, index s0 / 8
        // codes of slot s0 + r: a at position s0 + ch, b at position s0 - fh
        const int32_t wa = Codes::word_off(ch), wb = Codes::word_off(-fh);
        const uint32_t sha = Codes::bit_off(ch), shb = Codes::bit_off(-fh);
        int32_t runkey = INT32_MIN;             // max over chunks of (chunk max u) * 1024 + 1023 - chunk
        uint32_t fc = 0xffffffffu;              // first chunk with a live cell
        int32_t lc = -1;                        // last chunk with a live cell
        if (hlo <= hhi) {
#pragma unroll 1
            // the highest warp takes the first chunks of every pass: in a partial
            // last pass warp 0, which has the per-antidiagonal extra work (exact
            // extents, cell count, argmax) after the barrier, is the idle one
            for (int32_t c8w = c8base + 32 * (C::NW - 1 - warp); c8w <= c8last; c8w += C::NT) {
                const int32_t c8 = c8w + lane;
                const int32_t s0 = 8 * c8;
                const bool active = c8 <= c8last;
                const int32_t ri = (c8 & (C::SLOTS / 8 - 1)) * 4;  // word of slot s0
                const uint4 dw = *(const uint4 *)(cur + ri);  // d-2 (diag)
                const uint4 pw = *(const uint4 *)(oth + ri);  // d-1
                uint32_t nb;  // the neighbouring pair of d-1 beyond this chunk
                if (PAR) {
                    nb = __shfl_down_sync(0xffffffffu, pw.x, 1);
                    if (lane == 31) nb = oth[(ri + 4) & (C::WORDS - 1)];
                } else {
                    nb = __shfl_up_sync(0xffffffffu, pw.w, 1);
                    if (lane == 0) nb = oth[(ri - 1) & (C::WORDS - 1)];
                }
                Codes A, B;
                A.load(ca(), Codes::wstep() * c8 + wa, sha);  // slot s0 + r holds a_{s0 + r + ch}
                B.load(cb(), Codes::wstep() * c8 + wb, shb);  // and b_{fh - s0 - r}
                uint32_t mk[4];
                Codes::masks(A, B, mk);
                const uint32_t P4[4] = {pw.x, pw.y, pw.z, pw.w};
                const uint32_t D4[4] = {dw.x, dw.y, dw.z, dw.w};
                uint32_t U[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    uint32_t up, left;
                    if (PAR) {  // odd d: {E[s], E[s+1]}
                        left = P4[k];
                        up = prmt(P4[k], k < 3 ? P4[k + 1] : nb, 0x5432u);
                    } else {    // even d: {O[s-1], O[s]}
                        up = P4[k];
                        left = prmt(k > 0 ? P4[k - 1] : nb, P4[k], 0x5432u);
                    }
                    const uint32_t s2 = (mk[k] & smi2) | (~mk[k] & sma2);
                    const uint32_t t0 = __vimax3_s16x2(up, left, fg2);
                    const uint32_t dps = __viaddmax_s16x2(D4[k], s2, D16X2);
                    U[k] = vminu16(__viaddmax_s16x2(t0, gp2, dps), D16X2);  // exact kill
                }
                // slots outside [vlo, vhi] (band edges, cleared slots) are dead
                const int32_t rlo = vlo - s0, rhi = vhi - s0;
                if (rlo > 0 || rhi < 7) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t keep = ((2 * k >= rlo && 2 * k <= rhi) ? 0x0000ffffu : 0u) |
                                              ((2 * k + 1 >= rlo && 2 * k + 1 <= rhi) ? 0xffff0000u : 0u);
                        U[k] = (U[k] & keep) | (D16X2 & ~keep);
                    }
                }
                // (a lane past the range, s0 > hhi >= vhi, was masked dead above:
                // it must not store -- its slots may alias the far end of a wide
                // band -- but its dead chunk adds nothing to the reductions)
                if (active) *(uint4 *)(cur + ri) = make_uint4(U[0], U[1], U[2], U[3]);
                {
                    uint32_t cm2 = vmax16(__vimax3_s16x2(U[0], U[1], U[2]), U[3]);
                    cm2 = vmax16(cm2, prmt(cm2, cm2, 0x1032u));
                    const int32_t cm = sext_lo(cm2);  // the chunk's max u (D16 if all dead)
                    const int32_t crel = c8 - c8base;
                    runkey = max(runkey, cm * 1024 + (1023 - crel));
                    const int32_t v = crel | (cm >> 31);  // -1 if the chunk is dead
                    fc = min(fc, (uint32_t)v);
                    lc = max(lc, v);
                }
            }
        }

        // (5) antidiagonal reductions: warp CREDUX, one barrier, fold NW partials
        //     (one warp per task: the warp's CREDUX results are final, and a warp
        //     barrier orders the ring writes for the next antidiagonal)
        int32_t K, LC;
        uint32_t FC;
        {
            const int32_t K0 = __reduce_max_sync(0xffffffffu, runkey);
            const uint32_t FC0 = __reduce_min_sync(0xffffffffu, fc);
            const int32_t LC0 = __reduce_max_sync(0xffffffffu, lc);
            if constexpr (C::NW == 1) {
                K = K0; FC = FC0; LC = LC0;
                __syncwarp();
            } else {
                if (lane == 0) red(PAR)[warp] = make_int4(K0, (int32_t)FC0, LC0, 0);
                __syncthreads();
                // fold the NW partials: lane w reads warp w's (one LDS), CREDUX combines
                int4 r = make_int4(INT32_MIN, -1, -1, 0);
                if (lane < C::NW) r = red(PAR)[lane];
                K = __reduce_max_sync(0xffffffffu, r.x);
                FC = __reduce_min_sync(0xffffffffu, (uint32_t)r.y);
                LC = __reduce_max_sync(0xffffffffu, r.z);
            }
        }
        const bool h = LC >= 0;

        // (6) best after the complete antidiagonal, strict increase;
        //     warp 0 finds the argmax slot (first slot of the first chunk holding
        //     the max: the smallest i, c-amb-9)
        if (K >= 0) {
            const int32_t M = K >> 10;
            const int32_t V = M + Tc;
            if (V > t.best) {
                t.best = V;
                if (warp == C::ARG_WARP) {  // (warp 0 has the exact extents and the cell count)
                    const int32_t c = hbase + 8 * (1023 - (K & 1023));
                    const uint4 w = *(const uint4 *)(cur + ((c >> 1) & (C::WORDS - 1)));
                    const uint32_t W4[4] = {w.x, w.y, w.z, w.w};
                    int32_t r = 7;
#pragma unroll
                    for (int q = 7; q >= 0; --q) {
                        const int32_t u = (q & 1) ? sext_hi(W4[q >> 1]) : sext_lo(W4[q >> 1]);
                        if (u == M) r = q;
                    }
                    t.arg_i = c + r + ch;
                    t.arg_j = d - t.arg_i;
                }
            }
        }
        t.Tq[PAR] = Tc;
        t.Tn = t.best - P.xdrop;
        t.d = d;
        t.cF[PAR] = h ? hbase + 8 * (int32_t)FC : EMPTY_F;
        t.cL[PAR] = h ? hbase + 8 * LC + 7 : EMPTY_L;
        t.Dlo[PAR] = vlo <= vhi ? vlo : EMPTY_F;
        t.Dhi[PAR] = vlo <= vhi ? vhi : EMPTY_L;
        if (warp == 0) {  // exact live extents of d (for the cell count)
            int32_t F = EMPTY_F, L = EMPTY_L;
            if (h) {
                uint32_t l0, l1;
                chunk_live(PAR, t.cF[PAR], l0, l1);
                F = t.cF[PAR] + (l0 ? (__ffs(l0) - 1) >> 3 : 4 + ((__ffs(l1) - 1) >> 3));
                const int32_t cl = hbase + 8 * LC;
                chunk_live(PAR, cl, l0, l1);
                L = cl + (l1 ? 4 + ((31 - __clz(l1)) >> 3) : (31 - __clz(l0)) >> 3);
            }
            t.xF[PAR] = F;
            t.xL[PAR] = L;
        }

        // (7) termination: d and d-1 both empty (c-amb-7)
        if (t.cF[0] == EMPTY_F && t.cF[1] == EMPTY_F) return 1;
        // (8) the next antidiagonal touches at most the span of both arrays'
        //     written slots widened by 9 on each side: it must fit the ring
        const int32_t lo = min(t.Dlo[0], t.Dlo[1]), hi = max(t.Dhi[0], t.Dhi[1]);
        if (hi - lo + 1 > C::SLOTS - BAND_MARGIN) return 2;
        return 0;
    }
};

// Persistent kernel: each CTA pulls tasks (or hand-over records) from the
// level's list and sweeps them to the end; overflow goes to the next level.
template <int FMT, class C>
__global__ void __launch_bounds__(C::NT) k_band(const Params P, const LevelIO io) {
    __shared__ uint32_t s_pos;
    __shared__ int32_t s_arg[2];  // the argmax warp's result, for the writer (thread 0)
    BandCta<FMT, C> c;
    c.tid = threadIdx.x;
    c.lane = threadIdx.x & 31;
    c.warp = C::NW == 1 ? 0 : (int)(threadIdx.x >> 5);  // (a constant with one warp per task)
    const uint32_t count = *io.count;
    for (;;) {
        if (c.tid == 0) s_pos = atomicAdd(io.cursor, 1u);
        __syncthreads();
        const uint32_t pos = s_pos;
        __syncthreads();  // s_pos is rewritten for the next task
        if (pos >= count) return;
        const uint32_t task = io.list[pos];
        int rc = 2;
        if (P.xdrop <= BAND_XMAX) {
            const uint32_t rec = io.in_recs ? io.in_recs[pos] : NO_REC;
            if (rec != NO_REC) c.resume(P, io.rec_in + (size_t)rec * io.rec_in_stride);
            else c.init(P, task);
            if (io.stats && c.tid == 0)
                atomicAdd((unsigned long long *)&io.stats->tasks_started[io.level], 1ull);
            do {
                rc = (c.t.d & 1) ? c.template step<0>(P) : c.template step<1>(P);
            } while (rc == 0);
        }
        if (c.tid == 32 * C::ARG_WARP) { s_arg[0] = c.t.arg_i; s_arg[1] = c.t.arg_j; }
        __syncthreads();
        if (c.tid == 0) {
            if (rc == 1) {
                TaskRes tr;
                tr.best = c.t.best;
                tr.i = s_arg[0];
                tr.j = s_arg[1];
                tr.flags = 0;
                tr.cells = c.t.cells;
                io.tres[task] = tr;
                if (io.stats) {
                    atomicAdd((unsigned long long *)&io.stats->tasks_finished[io.level], 1ull);
                    atomicAdd((unsigned long long *)&io.stats->cells_per_level[io.level],
                              (unsigned long long)(c.t.cells - c.t.cells_entry));
                    atomicAdd((unsigned long long *)&io.stats->cells_total, (unsigned long long)c.t.cells);
                }
            } else {  // the CTA level restarts it from antidiagonal 0
                const uint32_t o = atomicAdd(io.out_count, 1u);
                io.out_list[o] = task;
            }
        }
        __syncthreads();  // warp 0's reads of this task's ring are done before the next init
    }
}

}  // namespace logan
