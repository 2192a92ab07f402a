"""Full-size parity in the launch shapes the benchmarks run.

Every BASELINE config at its full pair count (C4: 100K of its ~1M pairs),
through the C ABI, with the automatic level and shape choice -- the kernel
instantiation ``bench.py`` times for that config.  ``stats`` names the first
level's launch (level, window width, throughput / latency shape, in-kernel
helpers), so each case asserts WHICH instantiation it compared; the helpers
must have taken hand-overs when there were many.  1% of the pairs (every
100th) plus the 64 costliest pairs (the ones that escalate) are compared
element by element with the oracle; the per-pair cell counts must add up to
the device's total.
"""
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

# (config, X, pairs, first level, window width) -- the first level's kernel is
# k_window<G = W/32 (1 at level 1), R = 32 (w0 at level 1), FMT, next level's G, 32>
CASES = {
    "c3_x20": (3, 20, 100_000, 1, 32),     # k_window<1,32,2bit,2,32>
    "c3_x50": (3, 50, 100_000, 2, 64),     # k_window<2,32,2bit,4,32>
    "c3_x100": (3, 100, 100_000, 3, 128),  # k_window<4,32,2bit,8,32>
    "c2_x150": (2, 150, 100_000, 4, 256),  # k_window<8,32,2bit,16,32>
    "c2_x300": (2, 300, 20_000, 5, 512),   # k_window<16,32,2bit,32,32>
    "c2_x20": (2, 20, 100_000, 1, 32),     # k_window<1,32,2bit,2,32> (bench --config 2)
    "c4": (4, 50, 100_000, 2, 64),         # BELLA-like: spurious pairs escalate to 512 / 1024 / CTA
    "c5": (5, 100, 20_000, 3, 128),        # 50-100 kb reads
}


def _sample(b, w, stride=100, top=64):
    cost = (b.q_len.astype(np.int64) + b.t_len) - 2 * w.k
    idx = np.union1d(np.arange(0, b.n_pairs, stride), np.argsort(-cost, kind="stable")[:top])
    return idx


@pytest.mark.parametrize("case", list(CASES))
def test_full_size_launch_shape_parity(case):
    cfg, X, n, level, width = CASES[case]
    w = datagen.CONFIGS[cfg].with_(xdrop=X)
    b = datagen.generate(w, n_pairs=n, u8=False)
    db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
    st = logan.new_stats()
    out, cells = logan.xdrop_batch(db, w.match, w.mismatch, w.gap, X, stats=st)
    torch.cuda.synchronize()
    s = logan.stats_dict(st)
    assert (s["first_level"], s["first_width"], s["first_shape"], s["first_helpers"]) == \
        (level, width, "throughput", True), s
    overflowed = s["tasks_started"][level]  # tasks the next level (helpers or its launch) took
    if overflowed >= 16:
        assert s["helper_tasks"] > 0, s
    o, c = out.cpu().numpy(), cells.cpu().numpy().view(np.uint64)
    assert int(c.sum()) == s["cells_total"] and s["pairs_invalid"] == 0
    idx = _sample(b, w)
    ref_o, ref_c = oracle.pairs(b.pool_2bit, 1, b.q_off[idx], b.q_len[idx], b.t_off[idx], b.t_len[idx],
                                b.q_seed[idx], b.t_seed[idx], w.k, w.match, w.mismatch, w.gap, X,
                                pool_len=b.pool_len)
    bad = np.nonzero((o[idx] != ref_o).any(axis=1) | (c[idx] != ref_c))[0]
    assert len(bad) == 0, (f"{case}: {len(bad)} of {len(idx)} sampled pairs differ; first #{idx[bad[0]]}: "
                           f"gpu {o[idx[bad[0]]]} {c[idx[bad[0]]]} oracle {ref_o[bad[0]]} {ref_c[bad[0]]}")


@pytest.mark.parametrize("X", [20, 50, 100])
def test_config3_throughput_shape_forced_small_batch(X):
    """A C3 batch small enough for the automatic latency shape, forced into the
    throughput shape with helpers (options.flags bit 3): every pair exact."""
    w = datagen.CONFIGS[3].with_(xdrop=X)
    b = datagen.generate(w, n_pairs=600, u8=False)
    db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
    st = logan.new_stats()
    out, cells = logan.xdrop_batch(db, 1, -1, -1, X, stats=st, throughput_first=True)
    torch.cuda.synchronize()
    s = logan.stats_dict(st)
    assert s["first_shape"] == "throughput" and s["first_helpers"], s
    ref = oracle.pairs(b.pool_2bit, 1, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed, w.k, 1, -1, -1, X,
                       pool_len=b.pool_len)
    assert (out.cpu().numpy() == ref[0]).all() and (cells.cpu().numpy().view(np.uint64) == ref[1]).all()


def test_monotonicity_violation_counts_agree():
    """c-amb-16: a larger X can lower the score. Over the C3 X-sweep (and a
    burst-error variant, where extensions stop early) the number of pairs whose
    score drops from one X to the next must be the same on the GPU and in the
    oracle (SURVEY.md §8c c-amb-16: a statistical check, not an invariant)."""
    xs = (10, 20, 50, 100)
    for burst in (0.0, 0.5):
        w = datagen.CONFIGS[3].with_(burst=burst)
        b = datagen.generate(w, n_pairs=300, u8=False, pair_base=7000)
        db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
        g, r = [], []
        for X in xs:
            out, _ = logan.xdrop_batch(db, 1, -1, -1, X)
            torch.cuda.synchronize()
            g.append(out.cpu().numpy()[:, 0].astype(np.int64))
            ro, _ = oracle.pairs(b.pool_2bit, 1, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed, w.k,
                                 1, -1, -1, X, pool_len=b.pool_len)
            r.append(ro[:, 0].astype(np.int64))
        for a in range(len(xs) - 1):
            assert (g[a] == r[a]).all()
            assert int((g[a + 1] < g[a]).sum()) == int((r[a + 1] < r[a]).sum())
