"""Per-antidiagonal latency of one long task in each level shape (the critical path
of latency-bound runs: C5 shares, strong-scaling shares).

    python tools/latency_probe.py [--lib path]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2002_05200_b200 as logan  # noqa: E402

w = datagen.CONFIGS[5].with_(tlen_min=100000, tlen_max=100000)
b = datagen.generate(w, n_pairs=1)
# put the seed at the start so one extension covers the whole read pair
b.q_seed[:] = 0
b.t_seed[:] = 0
b.workload = b.workload.with_(k=0)
db = logan.to_device(b)
steps = int(b.q_len[0] + b.t_len[0])
for X in (20, 100):
    for lvl in (1, 2, 3, 4, 5, 6):
        for shape in ("latency", "throughput"):
            kw = dict(first_level=lvl, latency_first=shape == "latency", throughput_first=shape == "throughput")
            st = logan.new_stats()
            logan.xdrop_batch(db, 1, -1, -1, X, stats=st, **kw)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                logan.xdrop_batch(db, 1, -1, -1, X, **kw)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 3
            s = logan.stats_dict(st)
            print(f"X={X} level={lvl} shape={s['first_shape']}({s['first_width']}) ms={ms:.3f} "
                  f"ns/antidiagonal={1e6 * ms / steps:.1f} started={s['tasks_started']}", flush=True)
