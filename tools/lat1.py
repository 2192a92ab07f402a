"""Per-antidiagonal time of one long level-1 task (packed window) vs 32 such tasks in one warp."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2002_05200_b200 as logan  # noqa: E402

for npairs in (1, 16, 64, 256):
    w = datagen.CONFIGS[3].with_(tlen_min=20000, tlen_max=20000)
    b = datagen.generate(w, n_pairs=npairs)
    b.q_seed[:] = 0
    b.t_seed[:] = 0
    b.workload = b.workload.with_(k=0)
    db = logan.to_device(b)
    steps = int(max(b.q_len + b.t_len))
    kw = dict(first_level=1, throughput_first=True)
    st = logan.new_stats()
    logan.xdrop_batch(db, 1, -1, -1, 20, stats=st, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        logan.xdrop_batch(db, 1, -1, -1, 20, **kw)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    s = logan.stats_dict(st)
    print(f"{os.environ.get('LOGAN_LIB','default')[-12:]} pairs={npairs} (tasks {2*npairs}, {npairs} long) ms={ms:.3f} "
          f"ns/antidiagonal={1e6 * ms / steps:.1f} started={s['tasks_started'][:3]} shifts={s['window_shifts']}", flush=True)
