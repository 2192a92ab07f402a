// logan_xdrop.cu — C ABI and device pipeline of the B200 X-drop library.
//
// One call = (on the caller's stream, no host synchronisation):
//   1. k_expand   : validate pairs, split each into a left and a right
//                   extension task (Fig. 5), cost key m+n, a
//                   log-linear cost bucket per task; empty extensions are
//                   finished here (best 0 at (0,0), 0 cells)
//   2. k_scan     : bucket histogram -> descending start offsets
//   3. k_scatter  : tasks into a longest-first (LPT) work queue, the device
//                   counterpart of the paper's host load balancing
//   4. levels 1-6 : k_window<G, R> register-window sweeps, widening W = G*R
//                   from the level chosen for X; a task whose band outgrows a
//                   window is handed to the next level with its exact state
//   5. level 7    : k_band, one CTA per task, the band as int16 pairs in a
//                   shared-memory ring of 8192 slots (wide bands: large X)
//   6. level 8    : k_wide, one CTA per task, unbounded band (restart)
//   7. k_combine  : seed score + L + R -> logan_result_t, cells (c-amb-8/10)
#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "logan_impl.cuh"

namespace logan {
extern template LOGAN_RUN_BATCH_SIG(LOGAN_SEQ_U8);
extern template LOGAN_RUN_BATCH_SIG(LOGAN_SEQ_2BIT);
extern template LOGAN_RUN_BATCH_SIG(FMT_U8S);
extern template LOGAN_RUN_BATCH_SIG(LOGAN_SEQ_U8 | FMT_Z);
extern template LOGAN_RUN_BATCH_SIG(LOGAN_SEQ_2BIT | FMT_Z);
extern template LOGAN_RUN_BATCH_SIG(FMT_U8S | FMT_Z);
}  // namespace logan


using namespace logan;

extern "C" {

int logan_abi_version(void) { return LOGAN_ABI_VERSION; }

int logan_level_width(int32_t level, int32_t xdrop, int64_t max_ext_len, int32_t first_slots) {
    if (level == 1) return first_slots > 0 ? first_slots : auto_first_slots(xdrop, max_ext_len);
    if (level >= 2 && level <= NWIDTH - 1) return kWidth[level - 1];
    if (level == NWIDTH) return auto_top_width(xdrop);
    return 0;
}

const char *logan_strerror(int status) {
    switch (status) {
        case LOGAN_OK: return "ok";
        case LOGAN_EINVAL: return "invalid argument";
        case LOGAN_ECUDA: return "CUDA error";
        case LOGAN_ENOSPC: return "workspace too small";
        default: return "unknown status";
    }
}

size_t logan_workspace_bytes(int64_t n_pairs, int64_t max_ext_len) {
    if (n_pairs < 0 || max_ext_len < 0) return 0;
    return make_layout(n_pairs, max_ext_len).total;
}

static int check_args(const uint8_t *seq_pool, int32_t seq_fmt, int64_t pool_len, const void *q_off,
                      const void *q_len, const void *t_off, const void *t_len, const void *q_seed,
                      const void *t_seed, int64_t n_pairs, int32_t k, logan_scoring_t sc,
                      const logan_options_t *opt, const void *out) {
    if (n_pairs < 0 || n_pairs > ((int64_t)1 << 30)) return LOGAN_EINVAL;
    if (seq_fmt != LOGAN_SEQ_U8 && seq_fmt != LOGAN_SEQ_2BIT) return LOGAN_EINVAL;
    if (k < 0 || pool_len < 0) return LOGAN_EINVAL;
    const bool subst = opt && opt->subst;
    if (subst && (seq_fmt != LOGAN_SEQ_U8 || opt->alphabet < 1 || opt->alphabet > LOGAN_MAX_ALPHABET))
        return LOGAN_EINVAL;
    if (subst && (opt->flags & 32)) return LOGAN_EINVAL;  // SeqAn-compat: match / mismatch scoring only
    if (!subst && (sc.match <= 0 || sc.match > 127 || sc.mismatch >= 0 || sc.mismatch < -127))
        return LOGAN_EINVAL;
    if (sc.gap >= 0 || sc.gap < -127 || sc.xdrop < 0 || sc.xdrop > XDROP_MAX) return LOGAN_EINVAL;
    if (opt && (opt->flags & 4) && (opt->zdrop < 0 || opt->zdrop > XDROP_MAX)) return LOGAN_EINVAL;
    if (opt && (opt->first_level < 0 || opt->first_level > NLEVEL)) return LOGAN_EINVAL;
    if (opt && opt->first_slots != 0 && opt->first_slots != 16 && opt->first_slots != 20 && opt->first_slots != 24 &&
        opt->first_slots != 28 && opt->first_slots != 32)
        return LOGAN_EINVAL;
    if (n_pairs == 0) return LOGAN_OK;
    if (!seq_pool || !q_off || !q_len || !t_off || !t_len || !q_seed || !t_seed || !out) return LOGAN_EINVAL;
    if (((uintptr_t)seq_pool & 3) != 0) return LOGAN_EINVAL;
    return LOGAN_OK;
}

int logan_xdrop_batch(const uint8_t *seq_pool, int32_t seq_fmt, int64_t pool_len, const int64_t *q_off,
                      const int32_t *q_len, const int64_t *t_off, const int32_t *t_len, const int32_t *q_seed,
                      const int32_t *t_seed, int64_t n_pairs, int64_t max_ext_len, int32_t k, logan_scoring_t sc,
                      const logan_options_t *opt, logan_result_t *out, uint64_t *cells, logan_stats_t *stats,
                      void *workspace, size_t workspace_bytes, void *stream) {
    int st = check_args(seq_pool, seq_fmt, pool_len, q_off, q_len, t_off, t_len, q_seed, t_seed, n_pairs, k,
                        sc, opt, out);
    if (st != LOGAN_OK) return st;
    if (max_ext_len < 0 || max_ext_len >= ((int64_t)1 << 30)) return LOGAN_EINVAL;
    if (n_pairs == 0) return LOGAN_OK;
    if (!workspace || ((uintptr_t)workspace & 255) != 0) return LOGAN_EINVAL;
    // the caller's extension bound sizes the workspace (the CTA level's scratch)
    const Layout L = make_layout(n_pairs, max_ext_len);
    if (workspace_bytes < L.total) return LOGAN_ENOSPC;

    Params P;
    P.pool = (const uint32_t *)seq_pool;
    const int64_t bytes = seq_fmt == LOGAN_SEQ_2BIT ? (pool_len + 3) / 4 : pool_len;
    P.pool_words = (bytes + 3) / 4;
    if (P.pool_words < 1) P.pool_words = 1;
    P.pool_len = pool_len;
    P.q_off = q_off; P.q_len = q_len; P.t_off = t_off; P.t_len = t_len;
    P.q_seed = q_seed; P.t_seed = t_seed;
    P.n_pairs = n_pairs;
    P.max_ext = max_ext_len;
    P.k = k;
    P.match = sc.match; P.mismatch = sc.mismatch; P.gap = sc.gap;
    P.one = 1;
    P.poison = (opt && (opt->flags & 2)) ? 1 : 0;
    P.nopack = (opt && (opt->flags & 16)) ? 1 : 0;
    P.compat = (opt && (opt->flags & 32)) ? 1 : 0;
    P.subst = opt ? opt->subst : nullptr;
    P.alphabet = (opt && opt->subst) ? opt->alphabet : 0;
    P.stats = stats;
    P.info[0] = P.info[1] = P.info[2] = P.info[3] = 0;
    auto pk2h = [](int32_t v) { return ((uint32_t)v & 0xffffu) * 0x10001u; };
    P.gap2 = pk2h(sc.gap);
    P.fg2 = pk2h(-16384 - sc.gap);  // DEAD16 - gap (xdrop_window16.cuh)
    P.match2 = pk2h(sc.match);
    P.mis2 = pk2h(sc.mismatch);
    // X' = min(X, 4 max_ext w): no cell of any extension of the batch can drop
    // at or above that bound, so the results equal those at X (header, scoring)
    const int64_t w = P.subst ? 127 : std::max<int64_t>(sc.match, std::max<int64_t>(-sc.mismatch, -sc.gap));
    const int64_t xnp = 4 * std::max<int64_t>(max_ext_len, 1) * w;
    P.xdrop = (int32_t)std::min<int64_t>(sc.xdrop, xnp);
    // Z-drop fires only if best - M_d > Z, and best - M_d <= X' on any antidiagonal
    // with a live cell: Z >= X' is the same as no Z-drop (header, zdrop)
    P.zdrop = (opt && (opt->flags & 4) && opt->zdrop < P.xdrop) ? opt->zdrop : -1;
    // register windows keep X' <= 2^19 (argmax key range); beyond, the CTA level;
    // the SeqAn-compat mode is implemented on the CTA level only
    const bool wide_only = P.xdrop > WINDOW_XMAX || P.compat;

    cudaStream_t s = (cudaStream_t)stream;
    uint8_t *ws = (uint8_t *)workspace;
    if (P.zdrop >= 0) {  // the Z-drop builds of the kernels (FMT | FMT_Z)
        if (P.subst) return run_batch<FMT_U8S | FMT_Z>(P, opt, wide_only, out, cells, stats, ws, L, s);
        if (seq_fmt == LOGAN_SEQ_2BIT) return run_batch<LOGAN_SEQ_2BIT | FMT_Z>(P, opt, wide_only, out, cells, stats, ws, L, s);
        return run_batch<LOGAN_SEQ_U8 | FMT_Z>(P, opt, wide_only, out, cells, stats, ws, L, s);
    }
    if (P.subst) return run_batch<FMT_U8S>(P, opt, wide_only, out, cells, stats, ws, L, s);
    if (seq_fmt == LOGAN_SEQ_2BIT) return run_batch<LOGAN_SEQ_2BIT>(P, opt, wide_only, out, cells, stats, ws, L, s);
    return run_batch<LOGAN_SEQ_U8>(P, opt, wide_only, out, cells, stats, ws, L, s);
}

size_t logan_host_arena_bytes(int64_t n_pairs, int64_t pool_len, int32_t seq_fmt, int64_t max_ext_len) {
    if (n_pairs < 0 || pool_len < 0) return 0;
    const int64_t pool_bytes = seq_fmt == LOGAN_SEQ_2BIT ? (pool_len + 3) / 4 : pool_len;
    size_t o = 0;
    o += align256((size_t)pool_bytes + 16);
    o += 2 * align256(sizeof(int64_t) * (size_t)n_pairs);
    o += 4 * align256(sizeof(int32_t) * (size_t)n_pairs);
    o += align256(sizeof(logan_result_t) * (size_t)n_pairs);
    o += align256(sizeof(uint64_t) * (size_t)n_pairs);
    if (seq_fmt == LOGAN_SEQ_U8) o += align256(logan_pack_2bit_bytes(pool_len)) + 256;  // packed copy + n_other
    o += logan_workspace_bytes(n_pairs, max_ext_len);
    return o;
}

static int host_batch(const uint8_t *seq_pool, int32_t seq_fmt, int64_t pool_len, const int64_t *q_off,
                      const int32_t *q_len, const int64_t *t_off, const int32_t *t_len, const int32_t *q_seed,
                      const int32_t *t_seed, int64_t n_pairs, int32_t k, logan_scoring_t sc,
                      const logan_options_t *opt, logan_result_t *out, uint64_t *cells, void *device_arena,
                      size_t arena_bytes, void *stream, bool sync);

int logan_xdrop_batch_host(const uint8_t *seq_pool, int32_t seq_fmt, int64_t pool_len, const int64_t *q_off,
                           const int32_t *q_len, const int64_t *t_off, const int32_t *t_len,
                           const int32_t *q_seed, const int32_t *t_seed, int64_t n_pairs, int32_t k,
                           logan_scoring_t sc, const logan_options_t *opt, logan_result_t *out,
                           uint64_t *cells, void *device_arena, size_t arena_bytes, void *stream) {
    return host_batch(seq_pool, seq_fmt, pool_len, q_off, q_len, t_off, t_len, q_seed, t_seed, n_pairs, k, sc,
                      opt, out, cells, device_arena, arena_bytes, stream, true);
}

int logan_xdrop_batch_host_async(const uint8_t *seq_pool, int32_t seq_fmt, int64_t pool_len,
                                 const int64_t *q_off, const int32_t *q_len, const int64_t *t_off,
                                 const int32_t *t_len, const int32_t *q_seed, const int32_t *t_seed,
                                 int64_t n_pairs, int32_t k, logan_scoring_t sc, const logan_options_t *opt,
                                 logan_result_t *out, uint64_t *cells, void *device_arena, size_t arena_bytes,
                                 void *stream) {
    return host_batch(seq_pool, seq_fmt, pool_len, q_off, q_len, t_off, t_len, q_seed, t_seed, n_pairs, k, sc,
                      opt, out, cells, device_arena, arena_bytes, stream, false);
}

}  // extern "C"

// Copy-ahead (options.flags bit 6, asynchronous host calls): the inputs are copied
// on a library stream of the device as soon as the ARENA is free (its last call's
// results are out), not when `stream` reaches the call, so one compute stream with
// a ring of arenas overlaps every copy with the previous sweeps. Per-arena "free"
// events and one copy stream per device live for the process.
struct CopyAhead {
    cudaStream_t cs = nullptr;
    cudaEvent_t free_ev = nullptr, copied_ev = nullptr;
};
static int copy_ahead_for(const void *arena, CopyAhead &ca) {
    static std::mutex mu;
    static std::unordered_map<int, cudaStream_t> streams;
    static std::unordered_map<const void *, std::pair<cudaEvent_t, cudaEvent_t>> events;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return LOGAN_ECUDA;
    std::lock_guard<std::mutex> lk(mu);
    auto it = streams.find(dev);
    if (it == streams.end()) {
        cudaStream_t cs;
        if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return LOGAN_ECUDA;
        it = streams.emplace(dev, cs).first;
    }
    ca.cs = it->second;
    auto ie = events.find(arena);
    if (ie == events.end()) {
        cudaEvent_t a, b;
        if (cudaEventCreateWithFlags(&a, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&b, cudaEventDisableTiming) != cudaSuccess)
            return LOGAN_ECUDA;
        ie = events.emplace(arena, std::make_pair(a, b)).first;  // never recorded: waits return at once
    }
    ca.free_ev = ie->second.first;
    ca.copied_ev = ie->second.second;
    return LOGAN_OK;
}

static int host_batch(const uint8_t *seq_pool, int32_t seq_fmt, int64_t pool_len, const int64_t *q_off,
                      const int32_t *q_len, const int64_t *t_off, const int32_t *t_len, const int32_t *q_seed,
                      const int32_t *t_seed, int64_t n_pairs, int32_t k, logan_scoring_t sc,
                      const logan_options_t *opt, logan_result_t *out, uint64_t *cells, void *device_arena,
                      size_t arena_bytes, void *stream, bool sync) {
    int st = check_args(seq_pool, seq_fmt, pool_len, q_off, q_len, t_off, t_len, q_seed, t_seed, n_pairs, k,
                        sc, opt, out);
    if (st != LOGAN_OK) return st;
    if (n_pairs == 0) return LOGAN_OK;
    if (!device_arena || ((uintptr_t)device_arena & 255) != 0) return LOGAN_EINVAL;
    // the extension bound over the valid pairs (the same validation as the device's
    // k_expand; invalid pairs are rejected there whatever their lengths)
    int64_t max_ext = 0;
    for (int64_t p = 0; p < n_pairs; ++p) {
        const int64_t ql = q_len[p], tl = t_len[p], qs = q_seed[p], ts = t_seed[p];
        if (ql < 0 || tl < 0 || ql >= (1 << 30) || tl >= (1 << 30)) continue;
        if (qs < 0 || ts < 0 || qs + k > ql || ts + k > tl) continue;
        if (q_off[p] < 0 || t_off[p] < 0 || q_off[p] + ql > pool_len || t_off[p] + tl > pool_len) continue;
        max_ext = std::max(max_ext, std::max(std::max(qs, ts), std::max(ql - qs - k, tl - ts - k)));
    }
    const int64_t pool_bytes = seq_fmt == LOGAN_SEQ_2BIT ? (pool_len + 3) / 4 : pool_len;
    uint8_t *a = (uint8_t *)device_arena;
    size_t o = 0;
    uint8_t *d_pool = a + o;   o += align256((size_t)pool_bytes + 16);
    int64_t *d_qoff = (int64_t *)(a + o); o += align256(sizeof(int64_t) * (size_t)n_pairs);
    int64_t *d_toff = (int64_t *)(a + o); o += align256(sizeof(int64_t) * (size_t)n_pairs);
    int32_t *d_qlen = (int32_t *)(a + o); o += align256(sizeof(int32_t) * (size_t)n_pairs);
    int32_t *d_tlen = (int32_t *)(a + o); o += align256(sizeof(int32_t) * (size_t)n_pairs);
    int32_t *d_qs = (int32_t *)(a + o);   o += align256(sizeof(int32_t) * (size_t)n_pairs);
    int32_t *d_ts = (int32_t *)(a + o);   o += align256(sizeof(int32_t) * (size_t)n_pairs);
    logan_result_t *d_out = (logan_result_t *)(a + o); o += align256(sizeof(logan_result_t) * (size_t)n_pairs);
    uint64_t *d_cells = (uint64_t *)(a + o); o += align256(sizeof(uint64_t) * (size_t)n_pairs);
    uint8_t *d_pack = nullptr;
    uint64_t *d_other = nullptr;
    if (seq_fmt == LOGAN_SEQ_U8) {
        d_pack = a + o;                 o += align256(logan_pack_2bit_bytes(pool_len));
        d_other = (uint64_t *)(a + o);  o += 256;
    }
    if (o > arena_bytes) return LOGAN_ENOSPC;
    cudaStream_t s = (cudaStream_t)stream;
    const bool ahead = !sync && opt && (opt->flags & 64);
    CopyAhead ca;
    if (ahead) {
        st = copy_ahead_for(device_arena, ca);
        if (st != LOGAN_OK) return st;
        if (cudaStreamWaitEvent(ca.cs, ca.free_ev, 0) != cudaSuccess) return LOGAN_ECUDA;
    }
    cudaStream_t cs = ahead ? ca.cs : s;  // the inputs' stream
    const size_t n8 = sizeof(int64_t) * (size_t)n_pairs, n4 = sizeof(int32_t) * (size_t)n_pairs;
    if (cudaMemsetAsync(d_pool + pool_bytes, 0, 16, cs) != cudaSuccess) return LOGAN_ECUDA;
    if (cudaMemcpyAsync(d_pool, seq_pool, (size_t)pool_bytes, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
        cudaMemcpyAsync(d_qoff, q_off, n8, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
        cudaMemcpyAsync(d_toff, t_off, n8, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
        cudaMemcpyAsync(d_qlen, q_len, n4, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
        cudaMemcpyAsync(d_tlen, t_len, n4, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
        cudaMemcpyAsync(d_qs, q_seed, n4, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
        cudaMemcpyAsync(d_ts, t_seed, n4, cudaMemcpyHostToDevice, cs) != cudaSuccess)
        return LOGAN_ECUDA;
    if (ahead && (cudaEventRecord(ca.copied_ev, ca.cs) != cudaSuccess ||
                  cudaStreamWaitEvent(s, ca.copied_ev, 0) != cudaSuccess))
        return LOGAN_ECUDA;
    if (o + logan_workspace_bytes(n_pairs, max_ext) > arena_bytes) return LOGAN_ENOSPC;
    // the synchronous call re-encodes a u8 pool of A/C/G/T as 2-bit (logan_pack_2bit):
    // identical results, the packed first window; the choice reads n_other (one sync)
    const uint8_t *run_pool = d_pool;
    int32_t run_fmt = seq_fmt;
    if (sync && seq_fmt == LOGAN_SEQ_U8 && !(opt && opt->subst)) {
        uint64_t other = 1;
        st = logan_pack_2bit(d_pool, pool_len, d_qoff, d_qlen, d_toff, d_tlen, n_pairs, d_pack,
                             logan_pack_2bit_bytes(pool_len), d_other, stream);
        if (st != LOGAN_OK) return st;
        if (cudaMemcpyAsync(&other, d_other, sizeof other, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return LOGAN_ECUDA;
        if (other == 0) { run_pool = d_pack; run_fmt = LOGAN_SEQ_2BIT; }
    }
    st = logan_xdrop_batch(run_pool, run_fmt, pool_len, d_qoff, d_qlen, d_toff, d_tlen, d_qs, d_ts, n_pairs, max_ext,
                           k, sc, opt, d_out, d_cells, nullptr, a + o, arena_bytes - o, stream);
    if (st != LOGAN_OK) return st;
    if (cudaMemcpyAsync(out, d_out, sizeof(logan_result_t) * (size_t)n_pairs, cudaMemcpyDeviceToHost, s) !=
        cudaSuccess)
        return LOGAN_ECUDA;
    if (cells && cudaMemcpyAsync(cells, d_cells, sizeof(uint64_t) * (size_t)n_pairs, cudaMemcpyDeviceToHost, s) !=
                     cudaSuccess)
        return LOGAN_ECUDA;
    if (ahead && cudaEventRecord(ca.free_ev, s) != cudaSuccess) return LOGAN_ECUDA;  // the arena is free again
    if (sync && cudaStreamSynchronize(s) != cudaSuccess) return LOGAN_ECUDA;
    return LOGAN_OK;
}
