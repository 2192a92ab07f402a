"""Multi-GPU driver: a static cell-count-balanced partition of ONE batch + one gather.

The path shards by pair: the paper's host "divides the
sequences into different groups that are then assigned to the GPUs"
(§IV-C) and "collects and organizes the results".  Here:

* ``pair_costs``: the estimated cells of a pair (the work a GPU does for it):
  per extension of m x n bases, a homologous alignment runs along its diagonal
  to the end of the shorter sequence and at most ceil(X/|gap|) gap steps
  beyond, i.e. about A = min(m + n, 2 min(m, n) + 2 ceil(X/|gap|))
  antidiagonals, over a band of about min(X + 8, min(m, n) + 1) cells
  (the band of a true pair is X + a few slots wide).
  Dovetail overlaps of very different read lengths (config 4) are therefore
  costed by their overlap, not by their read lengths.  Unrelated (spurious)
  pairs are not predictable from lengths; their ~30% share is balanced by the
  law of large numbers over the LPT order.
* ``partition_lpt``: greedy longest-processing-time partition into G parts
  (deterministic; ties go to the lowest part index).  Results never depend on
  the partition (each pair is independent) -- tests assert it.
* ``run_sharded``: each rank of a process group runs its part (by default the
  CUDA path on its own device) and the per-pair results are gathered to every
  rank in the original pair order (one ``all_gather``; 28 B/pair).  No
  collective touches the DP itself.
* ``xdrop_multi``: the same from ONE process over several local devices
  (each device's part launched asynchronously, then one host-side gather).
"""
from __future__ import annotations

import heapq

import numpy as np


def pair_costs(q_len, t_len, q_seed, t_seed, k: int, xdrop: int = 20, gap: int = -1) -> np.ndarray:
    """Estimated band cells of every pair (0 for invalid pairs)."""
    ql, tl = np.asarray(q_len, np.int64), np.asarray(t_len, np.int64)
    qs, ts = np.asarray(q_seed, np.int64), np.asarray(t_seed, np.int64)
    valid = (qs >= 0) & (ts >= 0) & (qs + k <= ql) & (ts + k <= tl)
    tail = 2 * (-(-int(xdrop) // max(1, -int(gap))))
    cost = np.zeros(len(ql), np.int64)
    for m, n in ((qs, ts), (ql - qs - k, tl - ts - k)):
        m, n = np.maximum(m, 0), np.maximum(n, 0)
        short = np.minimum(m, n)
        antidiag = np.minimum(m + n, 2 * short + tail)
        cost += antidiag * np.minimum(int(xdrop) + 8, short + 1)
    return np.where(valid, cost, 0)


def partition_lpt(costs: np.ndarray, n_parts: int) -> list[np.ndarray]:
    """Greedy LPT: pairs by descending cost, each to the least-loaded part
    (each part's indices returned in ascending order)."""
    costs = np.asarray(costs, np.int64)
    order = np.lexsort((np.arange(len(costs)), -costs))  # cost desc, index asc
    heap = [(0, p) for p in range(n_parts)]
    parts: list[list[int]] = [[] for _ in range(n_parts)]
    for idx in order:
        load, p = heapq.heappop(heap)
        parts[p].append(int(idx))
        heapq.heappush(heap, (load + int(costs[idx]), p))
    return [np.sort(np.asarray(p, np.int64)) for p in parts]


def subset(batch, idx: np.ndarray):
    """The pairs ``idx`` of a datagen.Batch, sharing its pools."""
    import datagen
    return datagen.Batch(batch.workload, batch.pair_base, batch.q_off[idx], batch.q_len[idx],
                         batch.t_off[idx], batch.t_len[idx], batch.q_seed[idx], batch.t_seed[idx],
                         batch.pool_len, batch.pool_u8, batch.pool_2bit)


def _gpu_compute(sub, w, fmt, device):
    import torch

    from . import api
    db = api.to_device(sub, fmt, device=device)
    out, cells = api.xdrop_batch(db, w.match, w.mismatch, w.gap, w.xdrop)
    torch.cuda.synchronize(device)
    return out.cpu().numpy(), cells.cpu().numpy().view(np.uint64)


def _parts(batch, w, n_parts):
    costs = pair_costs(batch.q_len, batch.t_len, batch.q_seed, batch.t_seed, w.k, w.xdrop, w.gap)
    return partition_lpt(costs, n_parts)


def run_sharded(batch, w, group=None, compute=None, fmt: int = 1, device=None):
    """Partition ``batch`` over the ranks of ``group``, compute the local part and
    gather every pair's (result[5], cells) to all ranks in the original order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    parts = _parts(batch, w, world)
    mine = parts[rank]
    sub = subset(batch, mine)
    if compute is None:
        out, cells = _gpu_compute(sub, w, fmt, device)
    else:
        out, cells = compute(sub, w)
    n = batch.n_pairs
    if world == 1:
        return out, cells
    # fixed-size exchange: pad every part to the largest one
    cap = max(len(p) for p in parts)
    rec = np.zeros((cap, 8), np.int32)
    rec[:len(mine), 0:5] = out
    rec[:len(mine), 5:7] = np.asarray(cells, np.uint64).view(np.int32).reshape(-1, 2)
    rec[:len(mine), 7] = 1
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.from_numpy(rec).to(dev)
    gathered = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(gathered, t, group=group)
    return _scatter_back(n, parts, [g.cpu().numpy() for g in gathered])


def _scatter_back(n, parts, recs):
    full_out = np.zeros((n, 5), np.int32)
    full_cells = np.zeros(n, np.uint64)
    for idx, g in zip(parts, recs):
        full_out[idx] = g[:len(idx), 0:5]
        full_cells[idx] = np.ascontiguousarray(g[:len(idx), 5:7]).view(np.uint64).reshape(-1)
    return full_out, full_cells


def xdrop_multi(batch, w, devices, fmt: int = 1):
    """One process, several local GPUs: partition ``batch`` with the same LPT
    cost model, launch every device's part asynchronously on its own stream,
    then gather the results in the original pair order (host side).
    Returns (int32[n,5], uint64[n])."""
    import torch

    from . import api
    devices = [torch.device(d) for d in devices]
    parts = _parts(batch, w, len(devices))
    pending = []
    for dev, idx in zip(devices, parts):
        if len(idx) == 0:
            pending.append((dev, None, None))
            continue
        db = api.to_device(subset(batch, idx), fmt, device=dev)
        out, cells = api.xdrop_batch(db, w.match, w.mismatch, w.gap, w.xdrop,
                                     stream=torch.cuda.current_stream(dev))
        pending.append((dev, out, cells))
    recs = []
    for (dev, out, cells), idx in zip(pending, parts):
        rec = np.zeros((len(idx), 7), np.int32)
        if out is not None:
            torch.cuda.synchronize(dev)
            rec[:, 0:5] = out.cpu().numpy()
            rec[:, 5:7] = cells.cpu().numpy().view(np.int32).reshape(-1, 2)
        recs.append(rec)
    return _scatter_back(batch.n_pairs, parts, recs)
