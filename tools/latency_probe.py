"""Per-antidiagonal latency of one long task in each level shape (C5-like tail)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import datagen
import paper_2002_05200_b200 as logan

w = datagen.CONFIGS[5].with_(tlen_min=100000, tlen_max=100000)
b = datagen.generate(w, n_pairs=1)
# put the seed at the start so one extension covers the whole read pair
b.q_seed[:] = 0
b.t_seed[:] = 0
b.workload = b.workload.with_(k=0)
db = logan.to_device(b)
for X in (20, 100):
    for lvl in (1, 2, 3, 4, 5, 6):
        for lat in (False, True):
            st = logan.new_stats()
            logan.xdrop_batch(db, 1, -1, -1, X, first_level=lvl, latency_first=lat, stats=st)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out, cells = logan.xdrop_batch(db, 1, -1, -1, X, first_level=lvl, latency_first=lat)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            steps = int(b.q_len[0] + b.t_len[0])
            s = logan.stats_dict(st)
            print(f"X={X} level={lvl} latency={int(lat)} ms={ms:.3f} ns/antidiagonal={1e6 * ms / steps:.1f} "
                  f"started={s['tasks_started']}", flush=True)
