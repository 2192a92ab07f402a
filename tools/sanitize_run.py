"""Small batches through every level shape, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import datagen
import paper_2002_05200_b200 as logan

small = "--small" in sys.argv  # racecheck is very slow: a handful of pairs, 2-bit only
w = datagen.CONFIGS[4]
b = datagen.generate(w, n_pairs=6 if small else 60)
if small:
    b.q_len[:] = np.minimum(b.q_len, 1200)
    b.t_len[:] = np.minimum(b.t_len, 1200)
    b.q_seed[:] = np.minimum(b.q_seed, b.q_len - w.k)
    b.t_seed[:] = np.minimum(b.t_seed, b.t_len - w.k)
for fmt in ((logan.LOGAN_SEQ_2BIT,) if small else (logan.LOGAN_SEQ_2BIT, logan.LOGAN_SEQ_U8)):
    db = logan.to_device(b, fmt)
    for lvl, lat, ho in ((None, False, 0), (1, False, 0), (2, True, 0), (1, False, 6), (7, False, 0)):
        out, cells = logan.xdrop_batch(db, 1, -1, -1, 50, first_level=lvl, latency_first=lat, handover=ho)
        torch.cuda.synchronize()
        print(fmt, lvl, lat, ho, int(cells.sum()), flush=True)

# substitution matrices and Z-drop (FMT_U8S and FMT | FMT_Z builds)
M = torch.as_tensor(datagen.protein_matrix()).cuda()
pb = datagen.protein_pairs(6 if small else 40, len_lo=50, len_hi=400)
dpb = logan.to_device(pb, logan.LOGAN_SEQ_U8)
for lvl, z in ((None, None), (1, 10), (3, None), (8, 5)):
    out, cells = logan.xdrop_batch(dpb, 1, -1, -4, 40, first_level=lvl, subst=M, zdrop=z)
    torch.cuda.synchronize()
    print("subst", lvl, z, int(cells.sum()), flush=True)
db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
for lvl, z in ((None, 20), (2, 0), (8, 10)):
    out, cells = logan.xdrop_batch(db, 1, -1, -1, 50, first_level=lvl, zdrop=z)
    torch.cuda.synchronize()
    print("zdrop", lvl, z, int(cells.sum()), flush=True)
# first-window widths (one lane per task), with the overflow hand-over to level 2
for fs in (16, 20):
    for X in (5, 50):
        out, cells = logan.xdrop_batch(db, 1, -1, -1, X, first_level=1, first_slots=fs)
        torch.cuda.synchronize()
        print("slots", fs, X, int(cells.sum()), flush=True)
# the band level's second stage (bands wider than the one-warp 4096-slot ring) and the
# packed one-warp latency shapes (W = 128 / 256)
rng = np.random.default_rng(5)
L = 4200
base = "".join(rng.choice(list("ACGT"), L))
mut = list(base)
for p in rng.choice(L, 60, replace=False):
    mut[p] = "ACGT"[("ACGT".index(mut[p]) + 1) % 4]
wb = datagen.from_strings([(base, "".join(mut), 0, 0)], k=5)
dwb = logan.to_device(wb, logan.LOGAN_SEQ_2BIT)
st = logan.new_stats()
out, cells = logan.xdrop_batch(dwb, 1, -1, -1, 20000, first_level=7, stats=st)
torch.cuda.synchronize()
s = logan.stats_dict(st)
print("band stage 2", int(cells.sum()), s["tasks_started"][6], s["tasks_finished"][6], flush=True)
for lvl in (3, 4):
    out, cells = logan.xdrop_batch(db, 1, -1, -1, 100, first_level=lvl, latency_first=True)
    torch.cuda.synchronize()
    print("one-warp packed", lvl, int(cells.sum()), flush=True)
