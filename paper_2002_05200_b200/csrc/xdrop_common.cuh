// xdrop_common.cuh — shared device-side definitions of the B200 X-drop path.
//
// Product code (CUDA path). Shares nothing with oracle/.
// Citations: PAPER.md line numbers ("P:<line>"), readings "c-amb-N" of
// DESIGN.md §3.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "logan_xdrop.h"

namespace logan {

// ---------------------------------------------------------------------------
// Per-call parameters (passed by value to every kernel).
struct Params {
    const uint32_t *pool;   // pool viewed as 32-bit words
    int64_t pool_words;     // readable words
    int64_t pool_len;       // bases
    const int64_t *q_off;
    const int32_t *q_len;
    const int64_t *t_off;
    const int32_t *t_len;
    const int32_t *q_seed;
    const int32_t *t_seed;
    int64_t n_pairs;
    int64_t max_ext;        // the caller's bound on extension lengths (longer: invalid pair)
    logan_stats_t *stats;   // NULL or the caller's device statistics
    int32_t k;
    int32_t match, mismatch, gap, xdrop;
    int32_t one;  // = 1 at run time; opaque to the compiler (see Window::cell)
    int32_t poison;  // test knob (options.flags bit 1): fill shared staging buffers with garbage first
    int32_t nopack;  // test knob (options.flags bit 4): int32 first window instead of the packed one
    int32_t compat;  // options.flags bit 5: SeqAn-compat mode (readings c-amb-24/25; CTA level only)
    const int8_t *subst;  // NULL, or an alphabet x alphabet substitution matrix (device memory)
    int32_t alphabet;
    int32_t zdrop;        // Z-drop threshold (c-amb-19), < 0 = off
    uint32_t info[4];     // the first level's launch (k_expand copies it into stats)
    // packed int16-pair constants of the packed windows (xdrop_window16.cuh), set
    // on the host: both halves = gap, DEAD16 - gap, match, mismatch (mod 2^16)
    uint32_t gap2, fg2, match2, mis2;
};

// Result of one extension task (L or R of one pair), 24 bytes.
struct TaskRes {
    int32_t best;
    int32_t i, j;   // argmax cell, extension-local (c-amb-8/9)
    int32_t flags;  // bit0 = pair invalid
    uint64_t cells; // band cells (c-amb-14)
};

// Work list of one level: tasks in `list[0 .. *count)`, taken through
// `*cursor`; tasks that overflow the level's window go to `out_list`.
struct LevelIO {
    const uint32_t *list;
    const uint32_t *count;
    uint32_t *cursor;
    uint32_t *out_list;
    uint32_t *out_count;
    logan_stats_t *stats;
    int32_t level;
    TaskRes *tres;
    // launch-shape dispatch: run only if min_count <= *count < max_count
    uint32_t min_count, max_count;
    // hand-over records (NULL = restart tasks from scratch)
    const uint32_t *in_recs;     // per list entry: record index or NO_REC
    const int32_t *rec_in;
    int64_t rec_in_stride;       // ints per record
    uint32_t *out_recs;
    int32_t *rec_out;
    int64_t rec_out_stride;
    uint32_t rec_out_cap;
    uint32_t *rec_out_count;
    int32_t handover;            // test knob: force a hand-over every N antidiagonals (0 = off)
    // in-kernel escalation helpers (first level only)
    int32_t helpers;             // blocks whose last warp is a helper
    uint32_t workers;            // producer groups (non-helper groups) in the launch
    uint32_t *done;              // producer groups that finished
    int32_t is_helper;           // this IO drives in-kernel helpers (stats.helper_tasks)
    int32_t sms;                 // > 0: first level, static first round over this many SMs
};

constexpr uint32_t NO_TASK = 0xffffffffu;

// ---------------------------------------------------------------------------
// A task: the sequences of one extension in extension coordinates
// (Fig. 5): a_i, i = 1..m and b_j, j = 1..n, with
//   left  (side 0): a_i = q[qs - i],       b_j = t[ts - j]      (read backwards)
//   right (side 1): a_i = q[qs + k + i - 1], b_j = t[ts + k + j - 1]
struct SeqRef {
    int64_t base;  // pool position of index 1
    int32_t dir;   // +1 / -1
    int32_t len;
};

struct TaskDesc {
    SeqRef a, b;
    bool valid;    // pair passed validation
};

// A pair is valid iff its seed and reads lie inside the reads / pool and both
// extensions are at most the caller's declared bound max_ext long (header,
// logan_xdrop_batch); invalid pairs get the invalid result.
__device__ __forceinline__ bool pair_valid(const Params &P, int64_t p) {
    const int64_t qo = P.q_off[p], to = P.t_off[p];
    const int32_t ql = P.q_len[p], tl = P.t_len[p], qs = P.q_seed[p], ts = P.t_seed[p];
    const int64_t k = P.k;
    if (ql < 0 || tl < 0 || ql >= (1 << 30) || tl >= (1 << 30)) return false;
    if (qs < 0 || ts < 0 || qs + k > ql || ts + k > tl) return false;
    if (qo < 0 || to < 0 || qo + ql > P.pool_len || to + tl > P.pool_len) return false;
    if (qs > P.max_ext || ts > P.max_ext || ql - qs - k > P.max_ext || tl - ts - k > P.max_ext) return false;
    return true;
}

__device__ __forceinline__ TaskDesc task_desc(const Params &P, uint32_t task) {
    const int64_t p = task >> 1;
    const int side = task & 1;
    TaskDesc t;
    t.valid = pair_valid(P, p);
    const int64_t qo = P.q_off[p], to = P.t_off[p];
    const int32_t ql = P.q_len[p], tl = P.t_len[p], qs = P.q_seed[p], ts = P.t_seed[p];
    if (side == 0) {
        t.a = {qo + qs - 1, -1, qs};
        t.b = {to + ts - 1, -1, ts};
    } else {
        t.a = {qo + qs + P.k, +1, ql - qs - P.k};
        t.b = {to + ts + P.k, +1, tl - ts - P.k};
    }
    if (!t.valid) {
        t.a.len = 0;
        t.b.len = 0;
    }
    return t;
}

// ---------------------------------------------------------------------------
// Pool access. FMT = LOGAN_SEQ_2BIT: 16 bases per word, 2 bits each, LSB
// first; FMT = LOGAN_SEQ_U8: 4 bases per word, one byte each (little endian).
template <int FMT> struct PoolFmt;
template <> struct PoolFmt<LOGAN_SEQ_2BIT> {
    static constexpr int LOG_CPW = 4, BITS = 2;
    static constexpr uint32_t MASK = 3u;
};
template <> struct PoolFmt<LOGAN_SEQ_U8> {
    static constexpr int LOG_CPW = 2, BITS = 8;
    static constexpr uint32_t MASK = 0xffu;
};
// Internal format id: a u8 pool of symbol codes scored with a substitution
// matrix (options.subst). Same pool layout as LOGAN_SEQ_U8.
constexpr int FMT_U8S = 2;
template <> struct PoolFmt<FMT_U8S> : PoolFmt<LOGAN_SEQ_U8> {};
// FMT | FMT_Z: the same format with the Z-drop stop compiled in (c-amb-19);
// the plain formats carry no Z-drop code at all (register pressure).
constexpr int FMT_Z = 4;
template <> struct PoolFmt<LOGAN_SEQ_U8 | FMT_Z> : PoolFmt<LOGAN_SEQ_U8> {};
template <> struct PoolFmt<LOGAN_SEQ_2BIT | FMT_Z> : PoolFmt<LOGAN_SEQ_2BIT> {};
template <> struct PoolFmt<FMT_U8S | FMT_Z> : PoolFmt<LOGAN_SEQ_U8> {};
__host__ __device__ constexpr int fmt_base(int f) { return f & 3; }
__host__ __device__ constexpr bool fmt_z(int f) { return (f & FMT_Z) != 0; }

// Substitution table of the register windows (FMT_U8S), in shared memory:
// entry (a << 6) + b for codes a, b < 32 (a code is read modulo 32; entries
// beyond the alphabet are 0), row / column 32 = the past-the-end sentinels
// (-127: cells outside the matrix stay below every earlier best).
constexpr int SUBST_TAB_BYTES = (32 << 6) + 33 + 15;  // 2096, padded to 16
__device__ __forceinline__ void load_subst_tab(const Params &P, int8_t *tab, int tid, int nt) {
    for (int q = tid; q < SUBST_TAB_BYTES; q += nt) {
        const int a = q >> 6, b = q & 63;
        int8_t v = 0;
        if (a == 32 || b == 32) v = -127;
        else if (b < 32 && a < P.alphabet && b < P.alphabet) v = P.subst[a * P.alphabet + b];
        tab[q] = v;
    }
}

__device__ __forceinline__ uint32_t pool_word(const Params &P, int64_t wi) {
    wi = wi < 0 ? 0 : (wi >= P.pool_words ? P.pool_words - 1 : wi);
    return __ldg(P.pool + wi);
}

// Code of the base at pool position pos (no caching; blocking load).
template <int FMT>
__device__ __forceinline__ uint32_t pool_base(const Params &P, int64_t pos) {
    using F = PoolFmt<FMT>;
    const uint32_t w = pool_word(P, pos >> F::LOG_CPW);
    return (w >> (F::BITS * (uint32_t)(pos & ((1 << F::LOG_CPW) - 1)))) & F::MASK;
}

// a_idx / b_idx with a sentinel outside 1..len.
template <int FMT>
__device__ __forceinline__ uint32_t seq_at(const Params &P, const SeqRef &s, int32_t idx, uint32_t sent) {
    if (idx < 1 || idx > s.len) return sent;
    return pool_base<FMT>(P, s.base + (int64_t)s.dir * (idx - 1));
}

// A sequential reader over one extension sequence: next() returns the code of
// index `idx` (a sentinel outside 1..len) and moves to idx + 1. The word holding
// the next base and the word after it are kept in registers; crossing a word
// boundary shifts them down and issues the load of the following word, whose
// latency is hidden until the next boundary (16 bases later for 2-bit).
// The common path is a shift, a mask and two compares; word addresses are plain
// pointers (the ABI guarantees 16 readable bytes past the pool's end, so a
// forward prefetch never needs a bound; a backward one stops at the pool start).
// seek() repositions the reader anywhere (blocking loads; rare: task start,
// resume and window shifts).
template <int FMT>
struct Stream {
    using F = PoolFmt<FMT>;
    static constexpr int CPW = 1 << F::LOG_CPW;
    SeqRef s;
    const uint32_t *wp;  // word holding the base at index max(idx, 1)
    uint32_t cur;        // *wp
    uint32_t nxt;        // wp[dir] (prefetched)
    int32_t idx;         // extension index returned by the next next()
    int32_t sh;          // bit offset of that base inside cur
    int32_t nld;         // words that may still be prefetched beyond wp in direction dir
                         // (going backwards: the words above the pool start)

    __device__ __forceinline__ void seek(const Params &P, int32_t i) {
        idx = i;
        const int32_t c = (i < 1 || s.len <= 0) ? 1 : (i > s.len ? s.len : i);
        const int64_t pos = s.base + (int64_t)s.dir * (c - 1);
        const int64_t wi = pos >> F::LOG_CPW;
        sh = F::BITS * (int32_t)(pos & (CPW - 1));
        const int64_t wc = wi < 0 ? 0 : (wi >= P.pool_words ? P.pool_words - 1 : wi);
        wp = P.pool + wc;
        nld = s.dir < 0 ? (int32_t)(wc < (1 << 30) ? wc : (1 << 30)) : (1 << 30);
        cur = __ldg(wp);
        nxt = nld > 0 ? __ldg(wp + s.dir) : 0u;
    }

    // word boundary crossed: shift the prefetched word in, prefetch the next one
    // (going backwards, one crossing past the last base can put wp on the word
    // before the pool: never prefetch below the pool start)
    __device__ __forceinline__ void refill(const Params &P) {
        sh -= s.dir * 32;
        wp += s.dir;
        cur = nxt;
        --nld;
        nxt = nld > 0 ? __ldg(wp + s.dir) : 0u;
    }

    // next() for the hot loop: the same result and state, with the refill
    // predicated instead of branched (in a warp of independent tasks some lane
    // crosses a word boundary on most steps, so the branch was nearly always
    // taken by the warp) and the sentinel chosen by a select.
    __device__ __forceinline__ uint32_t next_fast(uint32_t sent) {
        const int32_t i = idx++;
        const bool in = (uint32_t)(i - 1) < (uint32_t)s.len;  // 1 <= i <= len
        const uint32_t c = (cur >> sh) & F::MASK;
        const int32_t nsh = sh + (in ? s.dir * F::BITS : 0);
        const bool need = (uint32_t)nsh >= 32u;
        sh = nsh & 31;
        const uint32_t *wn = wp + (need ? s.dir : 0);
        cur = need ? nxt : cur;
        nld -= need ? 1 : 0;
        const uint32_t ld = (need && nld > 0) ? 1u : 0u;
        uint32_t v = need ? 0u : nxt;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.global.nc.u32 %0, [%1];\n\t}"
                     : "+r"(v) : "l"(wn + s.dir), "r"(ld));
        nxt = v;
        wp = wn;
        return in ? c : sent;
    }

    __device__ __forceinline__ uint32_t next(const Params &P, uint32_t sent) {
        const int32_t i = idx++;
        if (i < 1 || i > s.len) return sent;  // before the start: parked at index 1
        const uint32_t c = (cur >> sh) & F::MASK;
        // advance (also past index len: at most one extra word, inside the pool's
        // 16-byte padding going forward, bounded by the pool start going back)
        sh += s.dir * F::BITS;
        if (__builtin_expect((uint32_t)sh >= 32u, 0)) refill(P);  // once per CPW bases
        return c;
    }
};

__device__ __forceinline__ int32_t ceil_half(int32_t d) { return (d + 1) >> 1; }
__device__ __forceinline__ int32_t floor_half(int32_t d) { return d >> 1; }

}  // namespace logan
