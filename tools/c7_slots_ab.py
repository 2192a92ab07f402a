"""A/B of the first-window width on the protein-like config 7 (device time of the whole call)."""
import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
import datagen, paper_2002_05200_b200 as logan
pb = datagen.protein_pairs(100_000)
db = logan.to_device(pb, logan.LOGAN_SEQ_U8)
M = torch.as_tensor(datagen.protein_matrix()).cuda()
ws = logan.make_workspace(pb.n_pairs, db.max_ext_len, "cuda")
for fs in (0, 16, 20, 24, 16, 20, 24):
    for _ in range(2):
        out, cells = logan.xdrop_batch(db, 1, -1, -4, 50, workspace=ws, subst=M, first_slots=fs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = logan.new_stats()
    e0.record()
    for _ in range(5):
        out, cells = logan.xdrop_batch(db, 1, -1, -4, 50, workspace=ws, subst=M, first_slots=fs)
    e1.record(); torch.cuda.synchronize()
    logan.xdrop_batch(db, 1, -1, -4, 50, workspace=ws, subst=M, first_slots=fs, stats=st); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    c = int(cells.sum().item())
    print(f"first_slots={fs}: {ms:.3f} ms, {c / ms / 1e6:.1f} GCUPS, started {logan.stats_dict(st)['tasks_started'][:3]}", flush=True)
