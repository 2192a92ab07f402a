"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Bit-exact on every integer output: score, q/t begin/end and the cell count
(SURVEY.md §8c P5).  Inputs are seeded synthetic workloads from ``datagen``;
expected values come only from ``oracle/``.
"""
import itertools
import random

import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2002_05200_b200 as logan  # noqa: E402
from paper_2002_05200_b200 import build as _build  # noqa: E402

_build.build()

FMTS = (logan.LOGAN_SEQ_2BIT, logan.LOGAN_SEQ_U8)


def gpu_run(batch, X, match=1, mismatch=-1, gap=-1, fmt=logan.LOGAN_SEQ_2BIT, first_level=None,
            stats=None):
    db = logan.to_device(batch, fmt)
    out, cells = logan.xdrop_batch(db, match, mismatch, gap, X, first_level=first_level, stats=stats)
    torch.cuda.synchronize()
    return out.cpu().numpy(), cells.cpu().numpy().view(np.uint64)


def oracle_run(batch, X, match=1, mismatch=-1, gap=-1, idx=None):
    b = batch
    sel = slice(None) if idx is None else idx
    return oracle.pairs(b.pool_u8, 0, b.q_off[sel], b.q_len[sel], b.t_off[sel], b.t_len[sel],
                        b.q_seed[sel], b.t_seed[sel], b.workload.k, match, mismatch, gap, X,
                        pool_len=b.pool_len)


def assert_same(o_gpu, c_gpu, o_ref, c_ref, what=""):
    bad = np.nonzero((o_gpu != o_ref).any(axis=1) | (c_gpu != c_ref))[0]
    if len(bad):
        p = bad[0]
        raise AssertionError(f"{what}: {len(bad)} mismatching pairs; first #{p}: gpu {o_gpu[p]} "
                             f"cells {c_gpu[p]} vs oracle {o_ref[p]} cells {c_ref[p]}")


def ext_batch(pairs_ab, k=0):
    """Extensions E(A, B) as pairs with a k=0 seed at (0,0): L empty, R = E(A, B)."""
    return datagen.from_strings([(a, b, 0, 0) for a, b in pairs_ab], k=k)


# --------------------------------------------------------------------------
def test_exhaustive_tiny_extensions_all_levels():
    strings = ["".join(s) for L in range(0, 6) for s in itertools.product("AC", repeat=L)]
    pairs = [(a, b) for a in strings for b in strings if a and b]
    b = ext_batch(pairs)
    for X in (0, 1, 2, 3, 5, 2 ** 19):
        ref = oracle_run(b, X)
        for lvl in (1, 2, 3, 4, 5, 6, 7, 8):
            got = gpu_run(b, X, first_level=lvl)
            assert_same(*got, *ref, what=f"X={X} level={lvl}")


@pytest.mark.parametrize("scoring", [(1, -1, -1), (2, -3, -1), (1, -2, -3), (3, -1, -2), (5, -4, -7)])
def test_random_pairs_scoring_and_x_sweep(scoring):
    rng = random.Random(hash(scoring) & 0xffff)
    pairs = []
    for _ in range(600):
        L = rng.randint(1, 300)
        a = "".join(rng.choice("ACGT") for _ in range(L))
        # a mutated copy (sub/ins/del) or an unrelated read
        if rng.random() < 0.7:
            bb = []
            for ch in a:
                r = rng.random()
                if r < 0.05:
                    bb.append(rng.choice("ACGT"))
                elif r < 0.1:
                    bb.append(ch + rng.choice("ACGT"))
                elif r < 0.15:
                    continue
                else:
                    bb.append(ch)
            b = "".join(bb) or "A"
        else:
            b = "".join(rng.choice("ACGT") for _ in range(rng.randint(1, 300)))
        k = rng.randint(0, min(len(a), len(b), 5))
        qs, ts = rng.randint(0, len(a) - k), rng.randint(0, len(b) - k)
        pairs.append((a, b, qs, ts))
    batch = datagen.from_strings(pairs, k=0)
    ma, mi, g = scoring
    for X in (0, 1, 4, 10, 25, 60, 200):
        ref = oracle_run(batch, X, ma, mi, g)
        for fmt in FMTS:
            got = gpu_run(batch, X, ma, mi, g, fmt=fmt)
            assert_same(*got, *ref, what=f"X={X} fmt={fmt} scoring={scoring}")


def test_adversarial_inputs():
    rng = random.Random(9)
    R = lambda n: "".join(rng.choice("ACGT") for _ in range(n))
    pairs = [
        ("A" * 500, "A" * 480, 100, 90),          # homopolymers
        ("AC" * 300, "AC" * 290, 50, 52),         # periodic repeats (seed off-phase)
        ("ACG" * 200, "ACG" * 210, 30, 33),
        (R(800), R(800), 400, 400),               # unrelated: wide bands
        (R(1500), R(1400), 10, 1390),             # unrelated, seed near opposite ends
        ("ACGT" * 100, "ACGT" * 100, 0, 0),       # seed at the start
        ("ACGT" * 100, "ACGT" * 100, 399, 399),   # seed at the end (k = 1)
        ("T" * 64, "G" * 64, 10, 10),             # disjoint alphabets
    ]
    batch = datagen.from_strings(pairs, k=1)
    for X in (0, 5, 20, 50, 100, 400):
        ref = oracle_run(batch, X)
        for lvl in (None, 1, 3, 5, 7, 8):
            for fmt in FMTS:
                got = gpu_run(batch, X, fmt=fmt, first_level=lvl)
                assert_same(*got, *ref, what=f"X={X} level={lvl} fmt={fmt}")


def test_invalid_and_empty_pairs():
    pairs = [("ACGTACGT", "ACGTACGT", 2, 2), ("ACGTACGT", "ACGTACGT", 0, 0),
             ("ACGTACGT", "ACGTACGT", 7, 7), ("ACGTACGT", "ACGTACGT", 5, 5)]
    b = datagen.from_strings(pairs, k=3)
    b.q_seed[2] = 7  # 7 + 3 > 8: invalid
    b.t_seed[3] = -1  # invalid
    got = gpu_run(b, 10)
    ref = oracle_run(b, 10)
    assert_same(*got, *ref)
    assert tuple(got[0][2]) == (-2 ** 31, -1, -1, -1, -1) and got[1][2] == 0
    # n_pairs = 0 is a no-op
    e = datagen.from_strings([], k=3)
    db = logan.to_device(e)
    out, cells = logan.xdrop_batch(db, 1, -1, -1, 10)
    assert out.numel() == 0


@pytest.mark.parametrize("X", [50])
def test_config1_all_pairs(X):
    b = datagen.generate(datagen.CONFIGS[1])
    ref = oracle_run(b, X)
    st = logan.new_stats()
    got = gpu_run(b, X, stats=st)
    assert_same(*got, *ref, what="C1")
    s = logan.stats_dict(st)
    assert s["cells_total"] == int(ref[1].sum())
    for fmt in FMTS:
        for lvl in (2, 3, 7, 8):
            got = gpu_run(b, X, fmt=fmt, first_level=lvl)
            assert_same(*got, *ref, what=f"C1 fmt={fmt} level={lvl}")


def test_config2_full_size_sampled():
    """Full C2 (100K pairs, X=20) in the launch configuration bench.py times;
    every 50th pair against the oracle, u8 == 2-bit on all pairs."""
    w = datagen.CONFIGS[2]
    b = datagen.generate(w)
    got = gpu_run(b, w.xdrop)
    idx = np.arange(0, b.n_pairs, 50)
    ref = oracle_run(b, w.xdrop, idx=idx)
    assert_same(got[0][idx], got[1][idx], *ref, what="C2 sample")
    got8 = gpu_run(b, w.xdrop, fmt=logan.LOGAN_SEQ_U8)
    assert (got8[0] == got[0]).all() and (got8[1] == got[1]).all()
    # invariants on every pair
    o = got[0]
    assert (o[:, 0] >= w.k).all() and (o[:, 1] <= b.q_seed).all() and (o[:, 2] <= b.q_len).all()
    assert (got[1] > 0).all()


@pytest.mark.parametrize("X", [5, 12, 18])
def test_config2_small_x_auto_widths_sampled(X):
    """Full C2 batch at the X values whose automatic first window is 16, 24 and
    28 slots, in the throughput shape with in-kernel helpers:
    every 100th pair against the oracle, and every pair equal to a run with
    the 32-slot first window (results never depend on the width)."""
    w = datagen.CONFIGS[2]
    b = datagen.generate(w)
    got = gpu_run(b, X)
    idx = np.arange(0, b.n_pairs, 100)
    ref = oracle_run(b, X, idx=idx)
    assert_same(got[0][idx], got[1][idx], *ref, what=f"C2 X={X} sample")
    db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
    out, cells = logan.xdrop_batch(db, 1, -1, -1, X, first_slots=32)
    torch.cuda.synchronize()
    assert (out.cpu().numpy() == got[0]).all() and (cells.cpu().numpy().view(np.uint64) == got[1]).all()


@pytest.mark.parametrize("X", [10, 20, 50, 100])
def test_config3_x_sweep_sampled(X):
    w = datagen.CONFIGS[3]
    b = datagen.generate(w, n_pairs=2000)
    got = gpu_run(b, X)
    idx = np.arange(0, b.n_pairs, 10)
    ref = oracle_run(b, X, idx=idx)
    assert_same(got[0][idx], got[1][idx], *ref, what=f"C3 X={X}")


def test_config4_bella_like_sampled():
    w = datagen.CONFIGS[4]
    b = datagen.generate(w, n_pairs=3000)
    st = logan.new_stats()
    got = gpu_run(b, w.xdrop, stats=st)
    idx = np.arange(0, b.n_pairs, 12)
    ref = oracle_run(b, w.xdrop, idx=idx)
    assert_same(got[0][idx], got[1][idx], *ref, what="C4")


def test_config5_long_reads_sampled():
    w = datagen.CONFIGS[5]
    b = datagen.generate(w, n_pairs=200)
    got = gpu_run(b, w.xdrop)
    idx = np.arange(0, b.n_pairs, 8)
    ref = oracle_run(b, w.xdrop, idx=idx)
    assert_same(got[0][idx], got[1][idx], *ref, what="C5")


def test_burst_errors_early_termination():
    w = datagen.CONFIGS[2].with_(burst=0.5, xdrop=20)
    b = datagen.generate(w, n_pairs=1500)
    got = gpu_run(b, 20)
    ref = oracle_run(b, 20)
    assert_same(*got, *ref, what="burst")


def test_host_entry_point_matches_device_entry():
    w = datagen.CONFIGS[1]
    b = datagen.generate(w, n_pairs=300)
    dev = gpu_run(b, w.xdrop)
    for fmt, pool in ((logan.LOGAN_SEQ_2BIT, b.pool_2bit), (logan.LOGAN_SEQ_U8, b.pool_u8)):
        arena = logan.HostArena(b.n_pairs, b.pool_len, fmt, b.max_ext_len())
        out, cells = logan.xdrop_batch_host(pool, fmt, b.pool_len, b.q_off, b.q_len, b.t_off,
                                            b.t_len, b.q_seed, b.t_seed, w.k, 1, -1, -1, w.xdrop,
                                            arena)
        assert (out == dev[0]).all() and (cells == dev[1]).all()


def test_host_copy_ahead_ring():
    """Asynchronous host calls with copy-ahead (options.flags bit 6): one stream, a
    ring of two arenas, eight steps over four DIFFERENT batches (an arena reused
    before its inputs are copied again would mix batches): every step's outputs
    equal the device entry point's on that batch."""
    w = datagen.CONFIGS[1]
    batches = [datagen.generate(w, n_pairs=400, pair_base=1000 * i) for i in range(4)]
    pool_len = max(b.pool_len for b in batches)
    ref = [gpu_run(b, w.xdrop) for b in batches]
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    hp = [[pin(x) for x in (b.pool_2bit, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed)] for b in batches]
    arenas = [logan.HostArena(400, pool_len, logan.LOGAN_SEQ_2BIT, max(b.max_ext_len() for b in batches))
              for _ in range(2)]
    outs = [np.zeros((400, 5), np.int32) for _ in range(8)]
    cells = [np.zeros(400, np.uint64) for _ in range(8)]
    s = torch.cuda.Stream()
    for step in range(8):
        b, h = batches[step % 4], hp[step % 4]
        logan.xdrop_batch_host(h[0], logan.LOGAN_SEQ_2BIT, b.pool_len, *h[1:], w.k, 1, -1, -1, w.xdrop,
                               arenas[step % 2], out=outs[step], cells=cells[step], stream=s,
                               asynchronous=True, copy_ahead=True)
    s.synchronize()
    for step in range(8):
        r = ref[step % 4]
        assert (outs[step] == r[0]).all() and (cells[step] == r[1]).all(), f"step {step}"


def test_repeatable_and_permutation_invariant():
    w = datagen.CONFIGS[1]
    b = datagen.generate(w, n_pairs=500)
    a1 = gpu_run(b, 50)
    a2 = gpu_run(b, 50)
    assert (a1[0] == a2[0]).all() and (a1[1] == a2[1]).all()
    perm = np.random.default_rng(1).permutation(b.n_pairs)
    bp = datagen.Batch(b.workload, 0, b.q_off[perm], b.q_len[perm], b.t_off[perm], b.t_len[perm],
                       b.q_seed[perm], b.t_seed[perm], b.pool_len, b.pool_u8, b.pool_2bit)
    ap = gpu_run(bp, 50)
    assert (ap[0] == a1[0][perm]).all() and (ap[1] == a1[1][perm]).all()


def _mixed_pairs(seed, n=300, maxlen=300):
    rng = random.Random(seed)
    pairs = []
    for _ in range(n):
        a = "".join(rng.choice("ACGT") for _ in range(rng.randint(1, maxlen)))
        if rng.random() < 0.6:
            b = "".join(ch if rng.random() > 0.12 else rng.choice(["", ch + rng.choice("ACGT"), rng.choice("ACGT")])
                        for ch in a) or "A"
        else:
            b = "".join(rng.choice("ACGT") for _ in range(rng.randint(1, maxlen)))
        pairs.append((a, b, rng.randint(0, len(a)), rng.randint(0, len(b))))
    return datagen.from_strings(pairs, k=0)


@pytest.mark.parametrize("lvl", [1, 2, 3, 4, 5, 6])
def test_latency_shapes_as_first_level(lvl):
    """Every level's latency shape (one warp per task), forced as the first level
    (at level 1 flags bit 0 selects the 32-slot window, the width that has one)."""
    b = _mixed_pairs(lvl)
    for X in (0, 3, 10, 30, 80):
        ref = oracle_run(b, X)
        for fmt in FMTS:
            db = logan.to_device(b, fmt)
            st = logan.new_stats()
            out, cells = logan.xdrop_batch(db, 1, -1, -1, X, first_level=lvl, latency_first=True, stats=st)
            torch.cuda.synchronize()
            s = logan.stats_dict(st)
            assert (s["first_level"], s["first_shape"], s["first_helpers"]) == (lvl, "latency", False), s
            assert_same(out.cpu().numpy(), cells.cpu().numpy().view(np.uint64), *ref,
                        what=f"latency level {lvl} X={X} fmt={fmt}")


@pytest.mark.parametrize("period", [2, 6, 40])
def test_forced_handover_is_exact(period):
    """Tasks handed over between levels every `period` antidiagonals (exact resume)."""
    b = _mixed_pairs(100 + period)
    for X in (0, 3, 10, 30):
        ref = oracle_run(b, X)
        for lvl in (1, 2):
            for lat in (False, True):
                db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
                out, cells = logan.xdrop_batch(db, 1, -1, -1, X, first_level=lvl, latency_first=lat,
                                               handover=period)
                torch.cuda.synchronize()
                assert_same(out.cpu().numpy(), cells.cpu().numpy().view(np.uint64), *ref,
                            what=f"handover {period} level {lvl} lat={lat} X={X}")


@pytest.mark.parametrize("fmt", FMTS)
def test_band_level_with_stale_shared_memory(fmt):
    """The band level's code buffers start as garbage (options.flags bit 1):
    stale codes of slots outside the staged range must not change the mismatch
    flags of the staged slots next to them (regression: a stale nibble > 8
    carried into its neighbour's flag, so an extension could miss its last
    cell depending on what an earlier kernel left in shared memory)."""
    for seed in (102, 106, 140):
        b = _mixed_pairs(seed)
        for X in (3, 10, 30):
            ref = oracle_run(b, X)
            for lvl, ho in ((1, 6), (2, 40), (6, 6), (7, 0)):
                db = logan.to_device(b, fmt)
                out, cells = logan.xdrop_batch(db, 1, -1, -1, X, first_level=lvl, latency_first=True,
                                               handover=ho, poison=True)
                torch.cuda.synchronize()
                assert_same(out.cpu().numpy(), cells.cpu().numpy().view(np.uint64), *ref,
                            what=f"poisoned band seed={seed} X={X} level {lvl} handover {ho} fmt={fmt}")


@pytest.mark.parametrize("X", [481, 560, 600, 680, 820])
def test_top_window_widths(X):
    """Level 6 runs 640-, 768- or 896-slot windows for 480 < X <= 820: as the
    automatic first level, forced hand-overs into and out of it (from the
    512-slot level, into the band level), and both pool formats."""
    w = datagen.CONFIGS[1].with_(xdrop=X)
    b = datagen.generate(w, n_pairs=24)
    ref = oracle_run(b, X)
    for fmt in FMTS:
        for lvl, ho in ((None, 0), (5, 0), (5, 60), (6, 40)):
            db = logan.to_device(b, fmt)
            out, cells = logan.xdrop_batch(db, 1, -1, -1, X, first_level=lvl, handover=ho)
            torch.cuda.synchronize()
            assert_same(out.cpu().numpy(), cells.cpu().numpy().view(np.uint64), *ref,
                        what=f"top window X={X} level {lvl} handover {ho} fmt={fmt}")


def test_mass_overflow_with_helpers():
    """Most tasks overflow the first window (X far above its width): helpers take
    what they can while level 1 runs (its throughput shape forced with
    options.flags bit 3: 8,000 tasks would otherwise take the latency shape),
    the next launch takes the rest; results exact."""
    w = datagen.CONFIGS[2].with_(xdrop=60)
    b = datagen.generate(w, n_pairs=4000)
    idx = np.arange(0, b.n_pairs, 10)
    ref = oracle_run(b, 60, idx=idx)
    st = logan.new_stats()
    db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
    out, cells = logan.xdrop_batch(db, 1, -1, -1, 60, first_level=1, stats=st, throughput_first=True)
    torch.cuda.synchronize()
    s = logan.stats_dict(st)
    assert (s["first_level"], s["first_shape"], s["first_helpers"]) == (1, "throughput", True), s
    assert s["tasks_started"][1] > 1000  # mass hand-over to the W=64 level
    assert s["helper_tasks"] > 0
    o, c = out.cpu().numpy(), cells.cpu().numpy().view(np.uint64)
    assert_same(o[idx], c[idx], *ref, what="mass overflow")


def test_cta_level_wide_bands():
    """The unbounded CTA level forced on BELLA-like pairs (spurious ones have
    bands of hundreds of slots: several cells per thread, many warps)."""
    w = datagen.CONFIGS[4]
    b = datagen.generate(w, n_pairs=40)
    b.q_len[:] = np.minimum(b.q_len, 2500)
    b.t_len[:] = np.minimum(b.t_len, 2500)
    b.q_seed[:] = np.minimum(b.q_seed, b.q_len - w.k)
    b.t_seed[:] = np.minimum(b.t_seed, b.t_len - w.k)
    ref = oracle_run(b, 50)
    for lvl in (8, 7, 6, None):
        got = gpu_run(b, 50, first_level=lvl)
        assert_same(*got, *ref, what=f"wide bands level={lvl}")


def test_cta_level_extension_equal_to_workspace_bound():
    """Regression: an extension exactly as long as max_ext_len must fit the CTA
    level's scratch (the workspace-size -> bound recovery once lost one base to
    alignment padding)."""
    w = datagen.CONFIGS[4]
    b = datagen.generate(w, n_pairs=6)
    b.q_len[:] = np.minimum(b.q_len, 1200)
    b.t_len[:] = np.minimum(b.t_len, 1200)
    b.q_seed[:] = np.minimum(b.q_seed, b.q_len - w.k)
    b.t_seed[:] = np.minimum(b.t_seed, b.t_len - w.k)
    assert b.max_ext_len() in set(b.q_seed.tolist()) | set(b.t_seed.tolist())
    ref = oracle_run(b, 50)
    for lvl in (8, None):
        got = gpu_run(b, 50, first_level=lvl)
        assert_same(*got, *ref, what=f"bound level={lvl}")


@pytest.mark.parametrize("slots", [16, 20, 24, 28, 32])
def test_first_window_widths(slots):
    """Every compiled first-window width (one lane per task) is exact, including
    the overflow hand-over to the next level: in the one-lane throughput shape
    with in-kernel helpers (forced: 300 pairs would pick the latency shape at 32
    slots) and in the automatic choice."""
    b = _mixed_pairs(300 + slots)
    # +1/-1/-1 takes the match - mismatch = 2 build of the packed window, (2, -3, -2) the general one
    for (ma, mi, g), X in itertools.product(((1, -1, -1), (2, -3, -2)), (0, 5, 12, 20)):
        ref = oracle_run(b, X, ma, mi, g)
        for tp in (True, False):
            db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
            st = logan.new_stats()
            out, cells = logan.xdrop_batch(db, ma, mi, g, X, first_level=1, first_slots=slots, stats=st,
                                           throughput_first=tp)
            torch.cuda.synchronize()
            s = logan.stats_dict(st)
            assert s["first_width"] == slots
            if tp:
                assert (s["first_shape"], s["first_helpers"]) == ("throughput", True), s
            assert_same(out.cpu().numpy(), cells.cpu().numpy().view(np.uint64), *ref,
                        what=f"first window {slots} X={X} scoring={(ma, mi, g)} throughput_first={tp}")


# --------------------------------------------------------------------------
# Ring level (level 7): one warp per task, the band in a shared-memory ring.

def _t2_pairs(n, cap, seed_off=0):
    """The paper's benchmark set (config 6: 2.5-7.5 kb reads, ~15% error),
    reads capped at `cap` bases so the oracle's full-band DP stays fast."""
    w = datagen.CONFIGS[6]
    b = datagen.generate(w, n_pairs=n, pair_base=seed_off)
    b.q_len[:] = np.minimum(b.q_len, cap)
    b.t_len[:] = np.minimum(b.t_len, cap)
    b.q_seed[:] = np.minimum(b.q_seed, b.q_len - w.k)
    b.t_seed[:] = np.minimum(b.t_seed, b.t_len - w.k)
    return b


@pytest.mark.parametrize("X", [150, 1000, 5000])
def test_ring_level_wide_x(X):
    """Large X (the paper's X sweep): bands of hundreds to thousands
    of slots, swept by the ring level; forced and automatic level choice, both
    pool formats, and the per-level statistics."""
    b = _t2_pairs(24, 3000)
    ref = oracle_run(b, X)
    for fmt in FMTS:
        for lvl in (7, None):
            st = logan.new_stats()
            got = gpu_run(b, X, fmt=fmt, first_level=lvl, stats=st)
            assert_same(*got, *ref, what=f"ring X={X} fmt={fmt} level={lvl}")
            s = logan.stats_dict(st)
            assert s["cells_total"] == int(ref[1].sum())
            if lvl == 7:
                assert s["tasks_finished"][6] == s["tasks_started"][6] > 0


def test_ring_level_resumes_window_records():
    """Tasks handed over by the widest register window (W = 1024) continue in
    the ring from the exact record: forced hand-overs after 2, 7 and 300
    antidiagonals, starting at level 6 (and at level 1, cascading through every
    window)."""
    b = _t2_pairs(16, 1500)
    for X in (60, 400, 3000):
        ref = oracle_run(b, X)
        for lvl, period in ((6, 2), (6, 7), (6, 300), (1, 2)):
            db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
            st = logan.new_stats()
            out, cells = logan.xdrop_batch(db, 1, -1, -1, X, first_level=lvl, handover=period, stats=st)
            torch.cuda.synchronize()
            assert_same(out.cpu().numpy(), cells.cpu().numpy().view(np.uint64), *ref,
                        what=f"ring resume X={X} level={lvl} period={period}")
            assert logan.stats_dict(st)["tasks_started"][6] > 0


def test_ring_overflow_and_large_x_go_to_cta_level():
    """A band wider than the ring (two 9 kb near-identical reads at a huge X)
    and X above the ring's int16 limit both end on the CTA level, exactly."""
    rng = np.random.default_rng(7)
    base = "".join(rng.choice(list("ACGT"), 9000))
    mut = list(base)
    for p in rng.choice(9000, 300, replace=False):
        mut[p] = "ACGT"[("ACGT".index(mut[p]) + 1) % 4]
    pairs = [(base, "".join(mut), 0, 0), (base[:3000], "".join(mut)[:3000], 1500, 1500)]
    b = datagen.from_strings(pairs, k=5)
    for X in (20000, 40000):
        ref = oracle_run(b, X)
        for lvl in (7, None):
            st = logan.new_stats()
            got = gpu_run(b, X, first_level=lvl, stats=st)
            assert_same(*got, *ref, what=f"ring overflow X={X} level={lvl}")
            s = logan.stats_dict(st)
            assert s["tasks_finished"][7] >= 1  # the 9 kb extension finished on the CTA level


def test_band_level_second_stage():
    """Bands between the first stage's 4096-slot ring and the second stage's 8192
    slots (two 6 kb near-identical reads at X = 20000: the band is the whole
    antidiagonal): the first stage restarts them on the second, which finishes
    them exactly; nothing reaches the CTA level. Both pool formats."""
    rng = np.random.default_rng(11)
    base = "".join(rng.choice(list("ACGT"), 6000))
    mut = list(base)
    for p in rng.choice(6000, 200, replace=False):
        mut[p] = "ACGT"[("ACGT".index(mut[p]) + 1) % 4]
    pairs = [(base, "".join(mut), 0, 0), (base[:2000], "".join(mut)[:2000], 1000, 1000)]
    b = datagen.from_strings(pairs, k=5)
    X = 20000
    ref = oracle_run(b, X)
    for fmt in FMTS:
        for lvl in (7, None):
            st = logan.new_stats()
            got = gpu_run(b, X, fmt=fmt, first_level=lvl, stats=st)
            assert_same(*got, *ref, what=f"band stage 2 fmt={fmt} level={lvl}")
            s = logan.stats_dict(st)
            assert s["tasks_finished"][7] == 0 and s["tasks_finished"][6] >= 1, s
            assert s["tasks_started"][6] > s["tasks_finished"][6], s  # a stage-1 restart


def test_band_level_restages_codes_on_long_reads():
    """Extensions much longer than the band level's staged code window (a 16384-
    position circular buffer, refilled when the band drifts out of it): 14 kb
    homologous reads at X = 300, forced onto level 7 and on the automatic
    path, both pool formats; burst insertions drift the band off the diagonal."""
    w = datagen.CONFIGS[3].with_(tlen_min=14000, tlen_max=14000, err=0.12, burst=0.3)
    b = datagen.generate(w, n_pairs=6, pair_base=11)
    for X in (300, 1500):
        ref = oracle_run(b, X)
        for fmt in FMTS:
            for lvl in (7, None):
                got = gpu_run(b, X, fmt=fmt, first_level=lvl)
                assert_same(*got, *ref, what=f"band restage X={X} fmt={fmt} level={lvl}")


# --------------------------------------------------------------------------
# Substitution-matrix scoring (P:381 protein alignment)

def _subst_run(b, M, gap, X, **kw):
    db = logan.to_device(b, logan.LOGAN_SEQ_U8)
    sub = torch.as_tensor(np.ascontiguousarray(M, dtype=np.int8)).cuda()
    out, cells = logan.xdrop_batch(db, 1, -1, gap, X, subst=sub, **kw)
    torch.cuda.synchronize()
    return out.cpu().numpy(), cells.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("X", [0, 10, 50, 200])
def test_subst_protein_pairs(X):
    """Protein-like pairs (20 codes, synthetic BLOSUM-shaped matrix), bit-exact
    against oracle.pairs_subst; includes a 30% share of unrelated pairs."""
    M = datagen.protein_matrix()
    b = datagen.protein_pairs(300, len_lo=50, len_hi=700, xdrop=X)
    rng = np.random.default_rng(X)
    unrel = rng.random(b.n_pairs) < 0.3  # pair an unrelated target with the query
    b.t_off = np.where(unrel, np.roll(b.t_off, 7), b.t_off)
    b.t_len = np.where(unrel, np.roll(b.t_len, 7), b.t_len).astype(np.int32)
    b.t_seed = np.where(unrel, np.minimum(np.roll(b.t_seed, 7), b.t_len - b.workload.k), b.t_seed).astype(np.int32)
    ref = oracle.pairs_subst(b.pool_u8, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed,
                             b.workload.k, M, -4, X, pool_len=b.pool_len)
    assert_same(*_subst_run(b, M, -4, X), *ref, what=f"protein subst X={X}")


def test_subst_matrix_equals_match_mismatch_path():
    """A DNA matrix M[a][b] = (a == b ? 1 : -1) on code pools gives the same
    results as the register-window path on the letter pool."""
    w = datagen.CONFIGS[1]
    b = datagen.generate(w, n_pairs=300)
    ref = gpu_run(b, 50, fmt=logan.LOGAN_SEQ_U8)
    codes = np.frombuffer(bytes.maketrans(b"ACGT", bytes([0, 1, 2, 3])), np.uint8)[b.pool_u8]
    bc = datagen.Batch(b.workload, 0, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed, b.pool_len, codes)
    M = [[1 if a == c else -1 for c in range(4)] for a in range(4)]
    assert_same(*_subst_run(bc, M, -1, 50), *ref, what="DNA matrix vs match/mismatch")


def test_subst_tiny_exhaustive_and_asymmetric():
    """Exhaustive short strings over 3 codes with an asymmetric matrix, several X."""
    M = [[2, -3, 1], [0, 4, -2], [-1, -1, 1]]
    strs = [bytes(s) for L in range(5) for s in itertools.product(range(3), repeat=L)]
    rng = random.Random(5)
    pairs = [(a, bb, 0, 0) for a in strs for bb in rng.sample(strs, 12)]
    b = datagen.from_strings(pairs, k=0)
    for X in (0, 2, 5, 1000):
        ref = oracle.pairs_subst(b.pool_u8, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed, 0, M, -2, X,
                                 pool_len=b.pool_len)
        assert_same(*_subst_run(b, M, -2, X), *ref, what=f"tiny subst X={X}")


@pytest.mark.parametrize("lvl", [1, 2, 3, 4, 5, 6, 7, 8])
def test_subst_every_level(lvl):
    """Substitution-matrix scoring forced onto every level (register windows 1-6
    with the shared-memory table, 7 = the band level which matrices skip, 8 = the
    CTA level), in both shapes and with forced hand-overs: bit-exact."""
    M = datagen.protein_matrix()
    b = datagen.protein_pairs(120, len_lo=40, len_hi=400, xdrop=40)
    for X in (0, 12, 40, 150):
        ref = oracle.pairs_subst(b.pool_u8, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed,
                                 b.workload.k, M, -4, X, pool_len=b.pool_len)
        for lat, ho in ((False, 0), (True, 0), (False, 6)):
            got = _subst_run(b, M, -4, X, first_level=lvl, latency_first=lat, handover=ho)
            assert_same(*got, *ref, what=f"subst level {lvl} lat={lat} handover {ho} X={X}")


# --------------------------------------------------------------------------
# Z-drop (c-amb-19; the X-drop variant the paper names)

@pytest.mark.parametrize("Z", [0, 3, 15, 60])
def test_zdrop_dna_every_level(Z):
    """Z-drop on DNA pairs (burst errors make it fire inside alignments),
    forced onto every level and both shapes, with hand-overs: bit-exact."""
    w = datagen.CONFIGS[1].with_(burst=0.5)
    b = datagen.generate(w, n_pairs=120)
    for X in (10, 40, 200):
        ref = oracle.pairs_z(b.pool_u8, 0, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed, w.k,
                             1, -1, -1, X, Z, pool_len=b.pool_len)
        for lvl, lat, ho in ((None, False, 0), (1, False, 0), (1, True, 6), (2, False, 40), (3, True, 0),
                             (6, False, 0), (7, False, 0), (8, False, 0)):
            for fmt in FMTS:
                db = logan.to_device(b, fmt)
                out, cells = logan.xdrop_batch(db, 1, -1, -1, X, first_level=lvl, latency_first=lat,
                                               handover=ho, zdrop=Z)
                torch.cuda.synchronize()
                assert_same(out.cpu().numpy(), cells.cpu().numpy().view(np.uint64), *ref,
                            what=f"zdrop Z={Z} X={X} level {lvl} lat={lat} ho={ho} fmt={fmt}")


def test_zdrop_with_substitution_matrix():
    M = datagen.protein_matrix()
    b = datagen.protein_pairs(150, len_lo=50, len_hi=500, xdrop=60)
    for X, Z in ((60, 10), (200, 40), (40, 0)):
        ref = oracle.pairs_z(b.pool_u8, 0, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed,
                             b.workload.k, 0, 0, -4, X, Z, subst=M, pool_len=b.pool_len)
        for lvl in (None, 1, 3, 8):
            got = _subst_run(b, M, -4, X, first_level=lvl, zdrop=Z)
            assert_same(*got, *ref, what=f"zdrop+subst X={X} Z={Z} level {lvl}")


def test_config7_and_zdrop_full_size_sampled():
    """Full-size runs of the f-4 modes in bench.py's launch configuration:
    config 7 (100K protein-like pairs, substitution matrix) and C2 with
    Z-drop; sampled pairs against the oracle, the cell totals against the
    per-pair sums, and Z-drop never exceeding the plain X-drop values."""
    M = datagen.protein_matrix()
    pb = datagen.protein_pairs(100_000)
    o, c = _subst_run(pb, M, -4, 50)
    idx = np.arange(0, pb.n_pairs, 97)
    ref = oracle.pairs_subst(pb.pool_u8, pb.q_off[idx], pb.q_len[idx], pb.t_off[idx], pb.t_len[idx],
                             pb.q_seed[idx], pb.t_seed[idx], pb.workload.k, M, -4, 50, pool_len=pb.pool_len)
    assert_same(o[idx], c[idx], *ref, what="C7 sample")
    w = datagen.CONFIGS[2]
    b = datagen.generate(w)
    db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
    out, cells = logan.xdrop_batch(db, 1, -1, -1, w.xdrop, zdrop=5)
    torch.cuda.synchronize()
    oz, cz = out.cpu().numpy(), cells.cpu().numpy().view(np.uint64)
    idx = np.arange(0, b.n_pairs, 97)
    refz = oracle.pairs_z(b.pool_u8, 0, b.q_off[idx], b.q_len[idx], b.t_off[idx], b.t_len[idx], b.q_seed[idx],
                          b.t_seed[idx], w.k, 1, -1, -1, w.xdrop, 5, pool_len=b.pool_len)
    assert_same(oz[idx], cz[idx], *refz, what="C2 Z-drop sample")
    plain = gpu_run(b, w.xdrop)
    assert (cz <= plain[1]).all() and (oz[:, 0] <= plain[0][:, 0]).all()


# --------------------------------------------------------------------------
# Boundary (ABI v2): the declared extension bound, X up to 2^28, Z >= X

def test_declared_extension_bound_rejects_longer_pairs_only():
    """A pair with an extension longer than the declared max_ext_len is an
    invalid pair (invalid result, 0 cells, counted in stats.pairs_invalid);
    every other pair keeps its exact result. Never a wrong result with OK."""
    import dataclasses
    w = datagen.CONFIGS[1]
    b = datagen.generate(w, n_pairs=200)
    ref_o, ref_c = oracle_run(b, w.xdrop)
    db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
    bound = 700
    ext = np.maximum(np.maximum(b.q_seed, b.t_seed),
                     np.maximum(b.q_len - b.q_seed - w.k, b.t_len - b.t_seed - w.k))
    over = ext > bound
    assert 0 < over.sum() < b.n_pairs
    st = logan.new_stats()
    out, cells = logan.xdrop_batch(dataclasses.replace(db, max_ext_len=bound), 1, -1, -1, w.xdrop, stats=st)
    torch.cuda.synchronize()
    o, c = out.cpu().numpy(), cells.cpu().numpy().view(np.uint64)
    assert logan.stats_dict(st)["pairs_invalid"] == int(over.sum())
    assert (o[over] == np.array([-2 ** 31, -1, -1, -1, -1])).all() and (c[over] == 0).all()
    assert (o[~over] == ref_o[~over]).all() and (c[~over] == ref_c[~over]).all()


def test_huge_x_runs_exactly():
    """X up to 2^28: X' = min(X, 4 max_ext w) gives the X = inf
    results; when X' > 2^19 (long extensions, large |w|) only the CTA level can
    hold it and the call runs there. Z >= X' is the same as no Z-drop."""
    w = datagen.CONFIGS[1]
    b = datagen.generate(w, n_pairs=40)
    for (ma, mi, g) in ((1, -1, -1), (100, -127, -127)):
        ref = oracle_run(b, 2 ** 28, ma, mi, g)
        st = logan.new_stats()
        got = gpu_run(b, 2 ** 28, ma, mi, g, stats=st)
        assert_same(*got, *ref, what=f"X=2^28 scoring {(ma, mi, g)}")
        s = logan.stats_dict(st)
        if 4 * b.max_ext_len() * max(ma, -mi, -g) > 2 ** 19:
            assert s["first_level"] == 8, s
        assert_same(*gpu_run(b, 2 ** 19, ma, mi, g), *ref, what="X=2^19 == X=2^28 here")
    db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
    ref = oracle_run(b, 30)
    out, cells = logan.xdrop_batch(db, 1, -1, -1, 30, zdrop=30)
    torch.cuda.synchronize()
    assert_same(out.cpu().numpy(), cells.cpu().numpy().view(np.uint64), *ref, what="Z >= X")


def test_partition_independence_multi_device_wrapper():
    """P4 partition independence: the single-process multi-device
    wrapper (multi.xdrop_multi) with G = 1, 2, 4, 8 parts -- all on cuda:0 here
    (this box has one GPU; the partition and gather logic is the same) --
    returns exactly the one-call results, pair by pair, for C1 and a BELLA-like
    C4 sample (dovetails + spurious pairs: the cost model's hard case)."""
    from paper_2002_05200_b200 import multi
    for cfg, n in ((1, 1000), (4, 600)):
        w = datagen.CONFIGS[cfg]
        b = datagen.generate(w, n_pairs=n, u8=False)
        ref = gpu_run(b, w.xdrop)
        for g in (1, 2, 4, 8):
            o, c = multi.xdrop_multi(b, w, ["cuda:0"] * g)
            assert_same(o, c, *ref, what=f"xdrop_multi config {cfg} G={g}")


@pytest.mark.parametrize("cfg,X,lvl", [(2, 5, None), (2, 12, None), (2, 20, None), (3, 20, None), (2, 60, 1),
                                       (6, 300, 1), (2, 20, 1), (2, 50, None), (2, 100, None), (6, 200, None),
                                       (6, 400, None), (4, 50, None), (2, 30, 2)])
def test_packed_first_window_equals_int32_window(cfg, X, lvl):
    """The packed int16 windows (2-bit pools, X <= 16000: level 1 and the
    throughput shapes of levels 2-5) against the int32 windows (options.flags
    bit 4) on every pair, and both against the oracle on a sample; a forced low
    first level at large X makes most tasks overflow (hand-over records written
    from and read into the packed layout)."""
    w = datagen.CONFIGS[cfg].with_(xdrop=X)
    b = datagen.generate(w, n_pairs=20000 if cfg != 3 else 4000, u8=False)
    db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
    res = []
    for nopack in (False, True):
        out, cells = logan.xdrop_batch(db, 1, -1, -1, X, first_level=lvl, nopack=nopack, throughput_first=True)
        torch.cuda.synchronize()
        res.append((out.cpu().numpy(), cells.cpu().numpy().view(np.uint64)))
    assert_same(*res[0], *res[1], what=f"packed vs int32 config {cfg} X={X} level={lvl}")
    idx = np.arange(0, b.n_pairs, 97)
    ref = oracle.pairs(b.pool_2bit, 1, b.q_off[idx], b.q_len[idx], b.t_off[idx], b.t_len[idx], b.q_seed[idx],
                       b.t_seed[idx], w.k, 1, -1, -1, X, pool_len=b.pool_len)
    assert_same(res[0][0][idx], res[0][1][idx], *ref, what=f"packed vs oracle config {cfg} X={X}")


# --------------------------------------------------------------------------
# SeqAn-compat mode (options.flags bit 5; readings c-amb-24/25, CTA level)

def test_compat_mode_matches_compat_oracle():
    """Bit-exact against oracle.pairs_compat: random tiny and adversarial
    pairs, C1, bursty C2 pairs (early drop-outs), with and without Z-drop."""
    rng = random.Random(31)
    pairs = []
    for _ in range(300):
        a = "".join(rng.choice("ACGT") for _ in range(rng.randint(1, 60)))
        bb = "".join(ch if rng.random() > 0.2 else rng.choice("ACGT") for ch in a) if rng.random() < 0.6 else \
            "".join(rng.choice("ACGT") for _ in range(rng.randint(1, 60)))
        pairs.append((a, bb, rng.randint(0, len(a)), rng.randint(0, len(bb))))
    batches = [datagen.from_strings(pairs, k=0), datagen.generate(datagen.CONFIGS[1], n_pairs=200),
               datagen.generate(datagen.CONFIGS[2].with_(burst=0.5), n_pairs=150)]
    for b in batches:
        for X in (0, 2, 10, 50):
            for Z in (None, 4):
                ref = oracle.pairs_compat(b.pool_u8, 0, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed,
                                          b.workload.k, 1, -1, -1, X, -1 if Z is None else Z, pool_len=b.pool_len)
                for fmt in FMTS:
                    db = logan.to_device(b, fmt)
                    st = logan.new_stats()
                    out, cells = logan.xdrop_batch(db, 1, -1, -1, X, compat=True, zdrop=Z, stats=st)
                    torch.cuda.synchronize()
                    assert logan.stats_dict(st)["first_level"] == 8
                    assert_same(out.cpu().numpy(), cells.cpu().numpy().view(np.uint64), *ref,
                                what=f"compat X={X} Z={Z} fmt={fmt}")


@pytest.mark.parametrize("lvl", [5, 6])
def test_packed_one_warp_shapes(lvl):
    """The packed one-warp shapes (32 lanes x 16 / 20..32 slots) as first level
    (latency shape) and with forced hand-overs, against the int32 ones and the
    oracle."""
    b = _mixed_pairs(500 + lvl, n=200, maxlen=600)
    for X in (3, 30, 120, 600):
        ref = oracle_run(b, X)
        for ho in (0, 6):
            res = []
            for nopack in (False, True):
                db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
                out, cells = logan.xdrop_batch(db, 1, -1, -1, X, first_level=lvl, latency_first=True, handover=ho,
                                               nopack=nopack)
                torch.cuda.synchronize()
                res.append((out.cpu().numpy(), cells.cpu().numpy().view(np.uint64)))
            assert_same(*res[0], *ref, what=f"packed one-warp level {lvl} X={X} ho={ho}")
            assert_same(*res[1], *ref, what=f"int32 one-warp level {lvl} X={X} ho={ho}")
