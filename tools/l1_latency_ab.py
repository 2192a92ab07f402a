"""A/B: level 1 (32-slot window) in its throughput shape (one lane per task, auto) against its
latency shape (one warp per task, options.flags bit 0) when a GPU holds few long tasks."""
import sys, torch
sys.path.insert(0, '/root/repo')
import datagen, paper_2002_05200_b200 as logan
for cfg, n, X in ((3, 3_000, 20), (3, 6_250, 20), (3, 12_500, 20), (3, 25_000, 20)):
    w = datagen.CONFIGS[cfg]
    b = datagen.generate(w, n_pairs=n, u8=False)
    db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
    ws = logan.make_workspace(n, db.max_ext_len, "cuda")
    base = None
    for lf in (False, True, False, True):
        for _ in range(2):
            out, cells = logan.xdrop_batch(db, 1, -1, -1, X, workspace=ws, latency_first=lf)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            out, cells = logan.xdrop_batch(db, 1, -1, -1, X, workspace=ws, latency_first=lf)
        e1.record(); torch.cuda.synchronize()
        res = (out.cpu().clone(), cells.cpu().clone())
        base = base or res
        same = torch.equal(base[0], res[0]) and torch.equal(base[1], res[1])
        ms = e0.elapsed_time(e1) / 3
        print(f"C{cfg} n={n} X={X} latency_first={lf}: {ms:.3f} ms, "
              f"{int(cells.sum().item()) / ms / 1e6:.1f} GCUPS same={same}", flush=True)
