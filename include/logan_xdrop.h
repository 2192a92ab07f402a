/*
 * logan_xdrop.h — C ABI v3 of the B200-native batched X-drop seed-and-extend
 * library (LOGAN, Zeni et al., arXiv 2002.05200).
 *
 * Citations are PAPER.md line numbers ("P:<line>") with the section, equation
 * or algorithm they fall in; "c-amb-N" refers to the numbered readings of the
 * paper listed in DESIGN.md §3.
 *
 * What one call computes (§III-A problem statement; Fig. 5 and
 * P:209 §IV-B seed split): for every (query, target, seed) pair
 *   - the LEFT extension  E(reverse q[0:qs), reverse t[0:ts))  and
 *   - the RIGHT extension E(q[qs+k:M), t[ts+k:N))
 * where E(A, B) is the X-drop antidiagonal sweep of Alg. 1 with
 * the cell rule of eq. P:85, the drop rule of P:89 (a cell with
 * S(i,j) < best - X is -inf and never considered again), `best` updated only
 * after an antidiagonal is complete and the band trimmed to the cells
 * that can still have a live predecessor (c-amb-6).
 * The pair result is
 *   score   = seed_score + best_L + best_R              (c-amb-10)
 *   q_begin = qs - i*_L,  q_end = qs + k + i*_R          ([begin, end), 0-based)
 *   t_begin = ts - j*_L,  t_end = ts + k + j*_R
 * where (i*, j*) is the cell at which each extension's best was FIRST reached
 * (smallest antidiagonal, then smallest query offset i; (0,0) if best = 0)
 * (c-amb-8, c-amb-9), and seed_score = sum_u (q[qs+u]==t[ts+u] ? match : mismatch).
 * `cells` counts, per extension, the interior cells of every antidiagonal band
 * [lo_d, hi_d] (DESIGN.md §3 "cell count"); the pair value is L + R.
 *
 * All arithmetic is int32; there is no floating point anywhere on the path.
 */
#ifndef LOGAN_XDROP_H
#define LOGAN_XDROP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LOGAN_ABI_VERSION 3

/* Linear scoring scheme (eq. P:85, read with signed addends, c-amb-2).
 * Requirements: 0 < match <= 127, -127 <= mismatch < 0, -127 <= gap < 0,
 * 0 <= xdrop <= 2^28. No cell of an extension with m + n bases
 * can ever drop once X >= 2 (m+n) w, w = max(match, -mismatch, -gap) (127 with
 * a substitution matrix): |S| <= (m+n) w and best <= (m+n) w, so best - X <= S.
 * The library therefore runs every call with X' = min(X, 4 max_ext_len w),
 * which gives results identical to X ("X = infinity" is any X >= that bound);
 * the register windows hold X' <= 2^19 (their argmax key u * 1027 + slot must
 * stay below 2^31), larger X' runs on the CTA level (int32 absolute scores). */
typedef struct {
    int32_t match;
    int32_t mismatch;
    int32_t gap;
    int32_t xdrop;
} logan_scoring_t;

/* Per-pair result, 20 bytes. Coordinates are 0-based half-open [begin, end)
 * in read coordinates. A pair whose seed or read range is invalid gets
 * {INT32_MIN, -1, -1, -1, -1}. */
typedef struct {
    int32_t score;
    int32_t q_begin;
    int32_t q_end;
    int32_t t_begin;
    int32_t t_end;
} logan_result_t;

/* Sequence pool formats.
 *  LOGAN_SEQ_U8   : one byte per base, bases compared by raw byte equality.
 *  LOGAN_SEQ_2BIT : A=0 C=1 G=2 T=3, four bases per byte, base b stored at
 *                   bits 2*(b mod 4) of byte floor(b/4) (LSB first). */
enum { LOGAN_SEQ_U8 = 0, LOGAN_SEQ_2BIT = 1 };

/* Status codes. */
enum {
    LOGAN_OK = 0,
    LOGAN_EINVAL = 1, /* bad scalar, null pointer or misaligned buffer */
    LOGAN_ECUDA = 2,  /* a CUDA launch or copy failed */
    LOGAN_ENOSPC = 3  /* workspace smaller than logan_workspace_bytes()  */
};

/* Options (may be passed as NULL = all defaults).
 *  first_level   : 0 = automatic from xdrop; 1..6 force the first
 *                  register-window level (windows of 32, 64, 128, 256, 512,
 *                  1024 diagonal slots; level 6 is 640 or 768 slots wide
 *                  when 480 < xdrop <= 680); 7 starts every task on the band
 *                  level (one CTA per task, the band as int16 pairs in an
 *                  8192-slot shared-memory ring; used for X <= 30000, wider
 *                  bands go on);
 *                  8 forces every task onto the unbounded CTA level.
 *                  Results never depend on it (tests assert this); only
 *                  speed does.
 *  timing_events : NULL, or LOGAN_N_STAGES * 2 cudaEvent_t created by the
 *                  caller (timing enabled). Event [2s] is recorded on `stream`
 *                  just before stage s and [2s+1] just after it, for every
 *                  stage the call launches: stage 0 = setup (task expansion,
 *                  LPT bucketing), stages 1..8 = levels 1..8, stage 9 =
 *                  combine. Stages not launched leave their events untouched.
 *  flags         : bit 0 = run the first level in its latency shape (one
 *                  warp per task) instead of its throughput shape; at level 1
 *                  this sets the first window to 32 slots (the only width
 *                  with a latency shape) unless first_slots forces another
 *                  width, in which case level 1 runs its one-lane shape
 *                  without in-kernel helpers.
 *                  bit 2 = Z-drop on, threshold `zdrop` (0 <= zdrop <= 2^28).
 *                  bit 3 = run the first level in its throughput shape even
 *                  when the batch has few tasks (test / tuning knob; bit 0 wins).
 *                  bit 5 = SeqAn-compat mode ([outside-PAPER]
 *                  readings c-amb-24/25 of DESIGN.md §3, not verified against
 *                  SeqAn): boundary cells (i = 0 or j = 0) on antidiagonals
 *                  d >= 2 are live only if S > best - X (strict), and each
 *                  extension's end cell is the "longest extension" -- the
 *                  best live cell (smallest i) of the last antidiagonal with a
 *                  live cell -- instead of the argmax; score = seed + best_L +
 *                  best_R as usual. Runs on the CTA level (8) only; match /
 *                  mismatch scoring only (a substitution matrix -> EINVAL).
 *                  bit 6 = copy-ahead (logan_xdrop_batch_host_async only):
 *                  the host inputs are copied on a library stream of the
 *                  device as soon as the device arena is free again (the
 *                  last call on that arena has written its results), instead
 *                  of when `stream` reaches this call; `stream` waits for the
 *                  copies before the sweep. One compute stream with a ring of
 *                  arenas then overlaps every step's copies with the previous
 *                  sweeps. The caller must not modify the host inputs after
 *                  the call until `stream` completes it (as without the flag)
 *                  and must not rely on earlier work on `stream` producing
 *                  them (they may be read before it runs). Ignored by the
 *                  synchronous entry point.
 *                  bit 4 = test / A-B knob: the first window of a 2-bit pool
 *                  runs on int32 values instead of packed int16 pairs.
 *                  bit 1 = test knob: the band level fills its shared-memory
 *                  code buffers with garbage before each task, so the tests
 *                  see the worst case of stale shared memory. Results never
 *                  depend on it.
 *  first_slots   : 0 = automatic; 16, 20, 24, 28 or 32 force the width of the
 *                  first window (one lane per task) when the first level is
 *                  level 1. Results never depend on it.
 *  handover      : test knob, 0 = off. If > 0, every task at a register
 *                  window level is handed over to the next level every
 *                  `handover` antidiagonals, exercising the exact hand-over.
 *                  Results never depend on it.
 *  zdrop         : with flags bit 2, the Z-drop stop (the X-drop variant the
 *                  paper names; reading c-amb-19): after
 *                  antidiagonal d, an extension ends if best - M_d > zdrop +
 *                  |gap| * |(i_d - i*) - (j_d - j*)|, M_d the largest live
 *                  score on d at (i_d, j_d) (smallest i), (i*, j*) the argmax
 *                  so far. X-drop pruning still applies. On an antidiagonal
 *                  with a live cell best - M_d <= X, so a Z >= X' never
 *                  fires and the library runs such calls without Z-drop
 *                  (identical results). Tasks with Z-drop
 *                  skip the band level (bands wider than the widest window
 *                  restart on the CTA level).
 *  subst, alphabet : substitution-matrix scoring (the
 *                  paper names protein alignment as future work).
 *                  NULL = match / mismatch. Otherwise a DEVICE pointer to an
 *                  int8 matrix of alphabet x alphabet entries, row-major,
 *                  1 <= alphabet <= 32, owned by the caller and read during
 *                  the call (both entry points): s(a_i, b_j) =
 *                  subst[a_i * alphabet + b_j] replaces "a_i == b_j ? match
 *                  : mismatch" in eq. P:85 and in the seed score; nothing
 *                  else changes. Requires seq_fmt = LOGAN_SEQ_U8 with every
 *                  base a code < alphabet (a code c is read as c mod 32 and
 *                  scores 0 against anything if that is >= alphabet);
 *                  scoring.match / .mismatch are then ignored (gap < 0 and
 *                  xdrop as usual). The register windows (levels 1-6) look
 *                  the score up in a shared-memory table; levels are chosen
 *                  from X / |gap|; there is no band level (7): bands wider
 *                  than the widest window go to the CTA level (8).
 */
#define LOGAN_N_STAGES 10
#define LOGAN_MAX_ALPHABET 32
typedef struct {
    int32_t first_level;
    int32_t flags;
    void *const *timing_events;
    int32_t handover;
    int32_t first_slots;
    const int8_t *subst;
    int32_t alphabet;
    int32_t zdrop;
    int64_t reserved[3];
} logan_options_t;

/* Per-call device-side statistics (optional output in DEVICE memory, may be
 * NULL; filled once the stream syncs): per level, the tasks that started
 * there, the tasks that finished there and their band cells; window shifts
 * summed over all tasks; the invalid pairs; and which kernel shape the first
 * level ran (diagnostics: tests assert which instantiation they exercised). */
typedef struct {
    uint64_t tasks_started[8];   /* entry l-1 = level l (1..8) */
    uint64_t tasks_finished[8];
    uint64_t cells_per_level[8];
    uint64_t window_shifts;
    uint64_t cells_total;
    uint64_t pairs_invalid;      /* pairs rejected by validation (see logan_xdrop_batch) */
    uint64_t helper_tasks;       /* tasks the first level's in-kernel helpers took */
    uint32_t first_level;        /* the level the call started on (1..8) */
    uint32_t first_width;        /* its register-window width in slots (0 for levels 7, 8) */
    uint32_t first_shape;        /* 0 = throughput shape (one lane or W/32 lanes per task), 1 = latency
                                    shape (one warp per task) */
    uint32_t first_helpers;      /* 1 if the first level ran in-kernel escalation helpers */
} logan_stats_t;

/* Bytes of device workspace a call with n_pairs pairs needs.
 * max_ext_len = the largest extension length (bases) on either side of any
 * seed, i.e. an upper bound on max(qs, ts, M-qs-k, N-ts-k); it sizes the
 * scratch of the unbounded CTA path. Returns 0 if n_pairs < 0. */
size_t logan_workspace_bytes(int64_t n_pairs, int64_t max_ext_len);

/*
 * logan_xdrop_batch — the whole hot path on one device, asynchronously on
 * `stream` (a cudaStream_t; NULL = legacy default stream).
 *
 * ALL pointers are DEVICE pointers owned by the caller; the library allocates
 * nothing, keeps no global state and is reentrant given distinct workspaces.
 *
 *  seq_pool   : the read pool, format `seq_fmt`, pool_len bases. The buffer
 *               must be 4-byte aligned and readable for 16 bytes past its last
 *               byte (the kernels load whole words and prefetch one ahead).
 *  q_off,t_off: int64[n_pairs] base offsets of query / target read in the pool
 *               (reads may be shared between pairs).
 *  q_len,t_len: int32[n_pairs] read lengths (bases), 0 <= len < 2^30.
 *  q_seed,t_seed: int32[n_pairs] seed start inside query / target read.
 *  max_ext_len: the caller's bound on every extension length (bases) of the
 *               batch: max over pairs of max(qs, ts, M-qs-k, N-ts-k), or any
 *               larger value, 0 <= max_ext_len < 2^30. It sizes the workspace
 *               (see logan_workspace_bytes) and picks the first window width;
 *               a pair with an extension longer than it is an INVALID pair
 *               (below), never a silently wrong result.
 *  k          : seed length (>= 0; k = 0 is a point seed).
 *  sc         : scoring and X.
 *  opt        : may be NULL (automatic).
 *  out        : logan_result_t[n_pairs] (device).
 *  cells      : uint64[n_pairs] (device) or NULL.
 *  stats      : logan_stats_t (device) or NULL.
 *  workspace  : device buffer of >= logan_workspace_bytes(n_pairs, max_ext_len)
 *               bytes, 256-byte aligned. Its contents are scratch.
 *
 * Errors: invalid scalars / NULL required pointers -> LOGAN_EINVAL and a
 * workspace smaller than logan_workspace_bytes(n_pairs, max_ext_len) ->
 * LOGAN_ENOSPC, both returned synchronously with nothing launched. A pair
 * whose ranges are invalid (q_seed < 0, q_seed + k > q_len, likewise for t, a
 * read outside [0, pool_len), or an extension longer than max_ext_len) gets
 * the invalid result {INT32_MIN, -1, -1, -1, -1} and cells = 0, and is counted
 * in stats->pairs_invalid; the rest of the batch is unaffected (device-side
 * validation cannot fail the call synchronously). A valid pair always gets its
 * exact result. A launch failure returns LOGAN_ECUDA. n_pairs = 0 is a no-op
 * returning LOGAN_OK.
 * Results are valid once `stream` has been synchronised.
 */
int logan_xdrop_batch(const uint8_t *seq_pool, int32_t seq_fmt, int64_t pool_len,
                      const int64_t *q_off, const int32_t *q_len,
                      const int64_t *t_off, const int32_t *t_len,
                      const int32_t *q_seed, const int32_t *t_seed,
                      int64_t n_pairs, int64_t max_ext_len, int32_t k, logan_scoring_t sc,
                      const logan_options_t *opt,
                      logan_result_t *out, uint64_t *cells, logan_stats_t *stats,
                      void *workspace, size_t workspace_bytes, void *stream);

/*
 * Host-buffer entry point (the end-to-end call): the same computation with
 * every input and output in HOST memory (pinned memory gives full-speed
 * copies). The caller provides one DEVICE arena of at least
 * logan_host_arena_bytes(...) bytes; the call copies the inputs into it
 * (host->device), runs logan_xdrop_batch on `stream`, copies `out` (and
 * `cells` if non-NULL) back (device->host) and synchronises `stream` before
 * returning. The extension bound is computed here from the host descriptors
 * (over the valid pairs), so no valid pair is ever rejected: an arena sized
 * for a smaller max_ext_len than the batch needs returns LOGAN_ENOSPC with
 * nothing launched. Same error behaviour as logan_xdrop_batch otherwise;
 * additionally returns LOGAN_ECUDA if a copy or the final synchronisation
 * fails.
 */
size_t logan_host_arena_bytes(int64_t n_pairs, int64_t pool_len, int32_t seq_fmt,
                              int64_t max_ext_len);
int logan_xdrop_batch_host(const uint8_t *seq_pool, int32_t seq_fmt, int64_t pool_len,
                           const int64_t *q_off, const int32_t *q_len,
                           const int64_t *t_off, const int32_t *t_len,
                           const int32_t *q_seed, const int32_t *t_seed,
                           int64_t n_pairs, int32_t k, logan_scoring_t sc,
                           const logan_options_t *opt,
                           logan_result_t *out, uint64_t *cells,
                           void *device_arena, size_t arena_bytes, void *stream);

/*
 * Asynchronous variant of logan_xdrop_batch_host: enqueues the host->device
 * copies, the sweep and the device->host copies on `stream` and returns without
 * synchronising; `out` / `cells` are valid once `stream` has been synchronised.
 * The host buffers must stay untouched until then (pinned memory makes the
 * copies truly asynchronous). With two arenas on two streams a caller overlaps
 * the copies of one batch with the sweep of the previous one.
 */
int logan_xdrop_batch_host_async(const uint8_t *seq_pool, int32_t seq_fmt, int64_t pool_len,
                                 const int64_t *q_off, const int32_t *q_len,
                                 const int64_t *t_off, const int32_t *t_len,
                                 const int32_t *q_seed, const int32_t *t_seed,
                                 int64_t n_pairs, int32_t k, logan_scoring_t sc,
                                 const logan_options_t *opt,
                                 logan_result_t *out, uint64_t *cells,
                                 void *device_arena, size_t arena_bytes, void *stream);

/*
 * logan_pack_2bit — device pre-pass: re-encode a LOGAN_SEQ_U8 pool whose bases
 * are the bytes 'A' 'C' 'G' 'T' (0x41 0x43 0x47 0x54) as a LOGAN_SEQ_2BIT pool
 * (A=0 C=1 G=2 T=3), asynchronously on `stream`. The sweep compares bases by
 * equality only (Alg. 1, the match / mismatch score of a
 * cell), so on such a pool logan_xdrop_batch gives bit-identical results for
 * the u8 pool and the packed one; the packed one runs the packed int16 first
 * window and moves a quarter of the bytes.
 *
 *  u8_pool     : device, pool_len bytes, 4-byte aligned, readable for 16
 *                bytes past its last byte (as seq_pool above). Not modified.
 *  q_off, q_len, t_off, t_len, n_pairs: the batch's read descriptors (device,
 *                as for logan_xdrop_batch); only the bytes inside these reads
 *                are checked (the sweep never compares any other byte). Pairs
 *                whose reads lie outside [0, pool_len) are skipped (they get
 *                the invalid result in either format).
 *  pool_2bit   : device, >= logan_pack_2bit_bytes(pool_len) bytes, 4-byte
 *                aligned, caller-owned: receives the (pool_len + 3) / 4 packed
 *                bytes followed by zero padding up to that size (so it meets
 *                seq_pool's 16-byte read-ahead rule).
 *  n_other     : device uint64 (8-byte aligned): set to the number of bytes
 *                outside {A, C, G, T} inside the reads. If it is non-zero the
 *                packed pool is NOT equivalent (the codes of other bytes are
 *                unspecified): keep the u8 pool. Read it after `stream` has
 *                been synchronised.
 * Errors: negative pool_len / n_pairs, NULL or misaligned pointers -> LOGAN_EINVAL; a
 * pool_2bit buffer smaller than logan_pack_2bit_bytes -> LOGAN_ENOSPC, both
 * synchronously with nothing launched; a launch failure -> LOGAN_ECUDA.
 *
 * logan_xdrop_batch_host (the synchronous host entry point) runs this pass
 * itself for a LOGAN_SEQ_U8 pool without a substitution matrix and takes the
 * packed pool when n_other == 0 (its arena includes the packed copy, see
 * logan_host_arena_bytes); the asynchronous variant never does (the choice
 * needs a host synchronisation).
 */
size_t logan_pack_2bit_bytes(int64_t pool_len);
int logan_pack_2bit(const uint8_t *u8_pool, int64_t pool_len, const int64_t *q_off, const int32_t *q_len,
                    const int64_t *t_off, const int32_t *t_len, int64_t n_pairs, uint8_t *pool_2bit,
                    size_t pool_2bit_bytes, uint64_t *n_other, void *stream);

/* Human-readable text for a status code (static storage). */
const char *logan_strerror(int status);

/* ABI version the library was built with (LOGAN_ABI_VERSION). */
int logan_abi_version(void);

/* Diagnostics (host only, no GPU needed): the diagonal-slot width of the
 * register window that level `level` (1..6) would run in a call with this
 * xdrop, max_ext_len (as for logan_workspace_bytes) and options.first_slots
 * (0 = automatic): level 1 is 16, 20, 24, 28 or 32 slots, levels 2..5 are 64,
 * 128, 256 and 512, level 6 is 640, 768, 896 or 1024. Returns 0 for levels
 * that are not register windows (7 = band level, 8 = CTA level) or out of
 * range. Results never depend on the widths; bench.py uses this to name the
 * kernel it reports. */
int logan_level_width(int32_t level, int32_t xdrop, int64_t max_ext_len, int32_t first_slots);

#ifdef __cplusplus
}
#endif

#endif /* LOGAN_XDROP_H */
