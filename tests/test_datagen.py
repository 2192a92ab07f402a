"""The seeded generator: determinism, shard independence, seed validity, shape."""
import numpy as np

import datagen


def test_deterministic_and_shardable():
    w = datagen.CONFIGS[1]
    a = datagen.generate(w, n_pairs=40)
    b = datagen.generate(w, n_pairs=40, n_threads=1)
    assert (a.q_len == b.q_len).all() and (a.pool_2bit == b.pool_2bit).all()
    # pairs [20, 40) generated alone equal the tail of the full batch
    c = datagen.generate(w, n_pairs=20, pair_base=20)
    for p in range(20):
        qa = datagen.decode_2bit(a.pool_2bit, a.q_off[20 + p], a.q_len[20 + p])
        qc = datagen.decode_2bit(c.pool_2bit, c.q_off[p], c.q_len[p])
        assert qa == qc
    assert (c.q_seed == a.q_seed[20:]).all() and (c.t_len == a.t_len[20:]).all()


def test_seeds_are_exact_kmers_and_formats_agree():
    for cfg in (1, 4):
        w = datagen.CONFIGS[cfg]
        b = datagen.generate(w, n_pairs=50 if cfg == 1 else 20)
        for p in range(b.n_pairs):
            q = datagen.decode_2bit(b.pool_2bit, b.q_off[p], b.q_len[p])
            t = datagen.decode_2bit(b.pool_2bit, b.t_off[p], b.t_len[p])
            assert bytes(b.pool_u8[b.q_off[p]:b.q_off[p] + b.q_len[p]]) == q
            qs, ts, k = b.q_seed[p], b.t_seed[p], w.k
            assert 0 <= qs and qs + k <= len(q) and 0 <= ts and ts + k <= len(t)
            assert q[qs:qs + k] == t[ts:ts + k]


def test_shapes_follow_the_recipe():
    w = datagen.CONFIGS[2]
    b = datagen.generate(w, n_pairs=300)
    # reads ~ template length (2.5 kb) with ~7.5% per-read error, indels balanced
    assert abs(b.q_len.mean() - 2500) < 40
    assert b.q_len.min() > 2300 and b.q_len.max() < 2700
    w4 = datagen.CONFIGS[4]
    b4 = datagen.generate(w4, n_pairs=400)
    assert 1000 <= b4.q_len.min() and b4.q_len.max() <= 2 * 30000 + 320
    lens = np.concatenate([b4.q_len, b4.t_len])
    # log-uniform on [1 kb, 30 kb]: median ~ sqrt(1000*30000) ~ 5.5 kb
    assert 3500 < np.median(lens) < 8000


def test_pack_roundtrip():
    s = "ACGTTGCAAC" * 7 + "G"
    p = datagen.pack_2bit(s)
    assert datagen.decode_2bit(p, 0, len(s)) == s.encode()
    assert datagen.decode_2bit(p, 3, 9) == s[3:12].encode()
