"""The u8 -> 2-bit device pre-pass (logan_pack_2bit, include/logan_xdrop.h).

The packed bytes are compared with datagen's host packer (the layout the
header fixes: base b at bits 2 (b mod 4) of byte b / 4), the other-byte count
with a numpy count, and the sweep on a packed u8 pool with the oracle.
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
from paper_2002_05200_b200 import _lib, build as _build  # noqa: E402

_build.build()
ACGT = np.frombuffer(b"ACGT", np.uint8)


def _pack(u8: np.ndarray, pool_len: int, shift: int = 0, reads=None):
    """Run logan_pack_2bit on u8[:pool_len] placed `shift` bytes into a device buffer;
    `reads` = [(q_off, q_len, t_off, t_len)] (default: one pair, both reads = the pool)."""
    lib = _lib.load()
    buf = torch.full((shift + len(u8) + 32,), ord("N"), dtype=torch.uint8, device="cuda")  # 'N' past the end
    buf[shift:shift + len(u8)] = torch.from_numpy(u8).cuda()
    if reads is None:
        reads = [(0, pool_len, 0, pool_len)] if pool_len else []
    r = np.array(reads, np.int64).reshape(-1, 4)
    qo, to = (torch.from_numpy(r[:, c].copy()).cuda() for c in (0, 2))
    ql, tl = (torch.from_numpy(r[:, c].astype(np.int32)).cuda() for c in (1, 3))
    nb = int(lib.logan_pack_2bit_bytes(pool_len))
    out = torch.full((nb,), 0xAB, dtype=torch.uint8, device="cuda")
    other = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    _lib.check(lib.logan_pack_2bit(buf.data_ptr() + shift, pool_len, qo.data_ptr(), ql.data_ptr(), to.data_ptr(),
                                   tl.data_ptr(), len(r), out.data_ptr(), nb, other.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return out.cpu().numpy(), int(other.item())


@pytest.mark.parametrize("shift", [0, 4, 8, 12])
@pytest.mark.parametrize("pool_len", [0, 1, 3, 4, 15, 16, 17, 31, 33, 1000, 4099, 1 << 16, (1 << 20) + 5])
def test_pack_equals_host_packer(pool_len, shift):
    rng = np.random.default_rng(pool_len * 7 + shift)
    u8 = ACGT[rng.integers(0, 4, pool_len)] if pool_len else np.zeros(0, np.uint8)
    got, other = _pack(u8, pool_len, shift)
    nbytes = (pool_len + 3) // 4
    exp = np.frombuffer(datagen.pack_2bit(u8.tobytes()), np.uint8)[:nbytes] if pool_len else np.zeros(0, np.uint8)
    assert other == 0
    assert (got[:nbytes] == exp).all()
    assert (got[nbytes:] == 0).all()  # the zero padding (and no stray bytes)
    if pool_len % 4:  # the codes past pool_len in the last byte are 0
        assert got[nbytes - 1] >> (2 * (pool_len % 4)) == 0


@pytest.mark.parametrize("shift", [0, 4])
def test_pack_counts_other_bytes_inside_reads(shift):
    rng = np.random.default_rng(5)
    n = 100_003
    u8 = ACGT[rng.integers(0, 4, n)]
    pos = rng.choice(n, 777, replace=False)
    u8[pos] = np.frombuffer(b"Nacgt\x00\x01\x02\x03-", np.uint8)[rng.integers(0, 10, 777)]
    _, other = _pack(u8, n, shift)
    assert other == 2 * 777  # both reads of the one pair cover the pool; 'N' past pool_len not counted
    # ragged reads (any byte offset / length), shared and invalid ones: the count is
    # the other bytes inside every valid read
    reads, exp = [], 0
    bad = np.zeros(n, bool)
    bad[pos] = True
    for _ in range(300):
        a, b = sorted(rng.integers(0, n, 2))
        c = int(rng.integers(0, n - 50))
        d = int(rng.integers(0, 50))
        reads.append((a, b - a, c, d))
        exp += int(bad[a:b].sum()) + int(bad[c:c + d].sum())
    reads.append((n - 3, 10, 0, 5))  # the query runs past the pool: the pair is skipped
    reads.append((-1, 4, 0, 5))
    assert _pack(u8, n, shift, reads)[1] == exp
    assert _pack(u8, n, shift, [(0, int(pos.min()), 0, 0)])[1] == 0


def test_xdrop_pack_u8_equals_oracle():
    w = datagen.CONFIGS[1]
    b = datagen.generate(w, n_pairs=400)
    ref = oracle.pairs(b.pool_u8, 0, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed, w.k, 1, -1, -1,
                       w.xdrop, pool_len=b.pool_len)
    db = logan.to_device(b, logan.LOGAN_SEQ_U8)
    for pack in (False, True):
        out, cells = logan.xdrop_batch(db, 1, -1, -1, w.xdrop, pack_u8=pack)
        torch.cuda.synchronize()
        assert (out.cpu().numpy() == ref[0]).all() and (cells.cpu().numpy().view(np.uint64) == ref[1]).all()


def test_other_bytes_keep_the_u8_path():
    # 'N' in both reads: raw byte equality (N == N matches) differs from any 2-bit
    # coding of the pool, so the pack must be refused and the u8 kernels run
    rng = np.random.default_rng(9)
    pairs = []
    for p in range(60):
        q = bytearray(ACGT[rng.integers(0, 4, 300)].tobytes())
        t = bytearray(q)
        for s in (q, t):
            for i in rng.choice(300, 12, replace=False):
                s[i] = ord("N")
        pairs.append((bytes(q), bytes(t), 100, 100))
    b = datagen.from_strings(pairs, k=17)
    ref = oracle.pairs(b.pool_u8, 0, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed, 17, 1, -1, -1, 30,
                       pool_len=b.pool_len)
    db = logan.to_device(b, logan.LOGAN_SEQ_U8)
    _, other = logan.pack_2bit(db)
    torch.cuda.synchronize()
    assert int(other.item()) == 60 * 24
    out, cells = logan.xdrop_batch(db, 1, -1, -1, 30, pack_u8=True)
    torch.cuda.synchronize()
    assert (out.cpu().numpy() == ref[0]).all() and (cells.cpu().numpy().view(np.uint64) == ref[1]).all()
    arena = logan.HostArena(b.n_pairs, b.pool_len, logan.LOGAN_SEQ_U8, b.max_ext_len())
    out_h, cells_h = logan.xdrop_batch_host(b.pool_u8, logan.LOGAN_SEQ_U8, b.pool_len, b.q_off, b.q_len, b.t_off,
                                            b.t_len, b.q_seed, b.t_seed, 17, 1, -1, -1, 30, arena)
    assert (out_h == ref[0]).all() and (cells_h == ref[1]).all()
