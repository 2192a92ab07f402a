"""A/B of the first-window width on C2 / C3 (X = 20): device time of the whole call."""
import sys, torch
sys.path.insert(0, '/root/repo')
import datagen, paper_2002_05200_b200 as logan
for cfg, n in ((2, 100_000), (3, 20_000)):
    w = datagen.CONFIGS[cfg]
    b = datagen.generate(w, n_pairs=n, u8=False)
    db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
    ws = logan.make_workspace(n, db.max_ext_len, "cuda")
    for fs in (0, 24, 28, 32, 24, 28):
        for _ in range(2):
            out, cells = logan.xdrop_batch(db, 1, -1, -1, w.xdrop, workspace=ws, first_slots=fs)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            out, cells = logan.xdrop_batch(db, 1, -1, -1, w.xdrop, workspace=ws, first_slots=fs)
        e1.record(); torch.cuda.synchronize()
        st = logan.new_stats()
        logan.xdrop_batch(db, 1, -1, -1, w.xdrop, workspace=ws, first_slots=fs, stats=st); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"C{cfg} first_slots={fs}: {ms:.3f} ms, {int(cells.sum().item()) / ms / 1e6:.1f} GCUPS, "
              f"started {logan.stats_dict(st)['tasks_started'][:3]}", flush=True)
