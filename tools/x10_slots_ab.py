"""A/B of the first-window width at small X (C6 templates 2.5-7.5 kb, C3 10 kb): device time of
the whole call, plus bit-equality of the outputs across widths (results never depend on it)."""
import sys, torch
sys.path.insert(0, '/root/repo')
import datagen, paper_2002_05200_b200 as logan
SETS = {"small": ((6, 100_000, (5, 8, 10, 12), (20, 16, 24, 20, 16)), (3, 50_000, (10,), (20, 16, 24, 20, 16))),
        "mid": ((6, 100_000, (14, 16, 18, 20), (24, 28, 32, 24, 28, 32)),
                (2, 100_000, (16, 18), (24, 28, 32, 24, 28, 32)))}
for cfg, n, xs, widths in SETS[sys.argv[1] if len(sys.argv) > 1 else "small"]:
    w = datagen.CONFIGS[cfg]
    b = datagen.generate(w, n_pairs=n, u8=False)
    db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
    ws = logan.make_workspace(n, db.max_ext_len, "cuda")
    for X in xs:
        base = None
        for fs in widths:
            for _ in range(2):
                out, cells = logan.xdrop_batch(db, 1, -1, -1, X, workspace=ws, first_slots=fs)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                out, cells = logan.xdrop_batch(db, 1, -1, -1, X, workspace=ws, first_slots=fs)
            e1.record(); torch.cuda.synchronize()
            st = logan.new_stats()
            logan.xdrop_batch(db, 1, -1, -1, X, workspace=ws, first_slots=fs, stats=st); torch.cuda.synchronize()
            res = (out.cpu().clone(), cells.cpu().clone())
            if base is None:
                base = res
            same = torch.equal(base[0], res[0]) and torch.equal(base[1], res[1])
            ms = e0.elapsed_time(e1) / 5
            print(f"C{cfg} X={X} first_slots={fs}: {ms:.3f} ms, {int(cells.sum().item()) / ms / 1e6:.1f} GCUPS, "
                  f"started {logan.stats_dict(st)['tasks_started'][:3]} same={same}", flush=True)
