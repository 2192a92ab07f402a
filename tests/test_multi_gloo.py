"""Multi-process host logic at world sizes 2 and 4 on CPU (gloo): partition + gather.

The per-rank compute is injected (the oracle stands in for the GPU here, as
the tests may use it); the CUDA path is the default compute on GPU boxes.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import datagen
from paper_2002_05200_b200 import multi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partition_is_a_balanced_permutation():
    w = datagen.CONFIGS[4]
    b = datagen.generate(w, n_pairs=3000, u8=False)
    costs = multi.pair_costs(b.q_len, b.t_len, b.q_seed, b.t_seed, w.k)
    for g in (1, 2, 4, 8):
        parts = multi.partition_lpt(costs, g)
        allidx = np.sort(np.concatenate(parts))
        assert (allidx == np.arange(b.n_pairs)).all()
        loads = np.array([costs[p].sum() for p in parts])
        assert loads.max() - loads.min() <= costs.max()  # LPT bound
        assert multi.partition_lpt(costs, g)[0].tolist() == parts[0].tolist()  # deterministic


def test_cost_model_follows_the_overlap():
    """A dovetail pair is costed by its overlap (the sweep ends about X/|gap|
    antidiagonals past the shorter sequence), not by its read lengths; equal
    extensions cost antidiagonals x band; invalid pairs cost 0."""
    k, X = 17, 50
    # seed in the middle of a 1 kb read against a 30 kb read: each side min 500
    c = multi.pair_costs([1000, 30000, 1000, 10], [30000, 30000, 1000, 10], [491, 15000, 491, 5],
                         [15000, 15000, 491, 20], k, X, -1)
    assert c[3] == 0
    # pair 0, left: min(491, 15000) = 491 -> min(15491, 2*491 + 2*50) = 1082 antidiagonals x 58;
    # right: min(492, 14983) = 492 -> 1084 x 58
    assert c[0] == 1082 * 58 + 1084 * 58
    # pair 2 (1 kb x 1 kb): the whole matrix, 982 and 984 antidiagonals x 58
    assert c[2] == 982 * 58 + 984 * 58
    assert c[0] < c[1] / 10  # the 1 kb x 30 kb pair is not costed like two 30 kb reads


def _oracle_compute(sub, w):
    import oracle
    return oracle.pairs(sub.pool_u8, 0, sub.q_off, sub.q_len, sub.t_off, sub.t_len, sub.q_seed,
                        sub.t_seed, w.k, w.match, w.mismatch, w.gap, w.xdrop, pool_len=sub.pool_len,
                        n_threads=2)


def _worker(rank, world, port, ret, cfg, n):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = datagen.CONFIGS[cfg]
    b = datagen.generate(w, n_pairs=n)
    out, cells = multi.run_sharded(b, w, compute=_oracle_compute)
    ret[rank] = (out.copy(), cells.copy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg,n", [(2, 1, 120), (4, 1, 90), (4, 4, 24)])
def test_sharded_gather_equals_single_process(world, cfg, n):
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), ret, cfg, n), nprocs=world, join=True)
    w = datagen.CONFIGS[cfg]
    b = datagen.generate(w, n_pairs=n)
    ref = _oracle_compute(b, w)
    for r in range(world):
        out, cells = ret[r]
        assert (out == ref[0]).all() and (cells == ref[1]).all()
