import sys
import numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import datagen, oracle
import paper_2002_05200_b200 as logan
w = datagen.CONFIGS[4]
b = datagen.generate(w, n_pairs=40)
b.q_len[:] = np.minimum(b.q_len, 2500); b.t_len[:] = np.minimum(b.t_len, 2500)
b.q_seed[:] = np.minimum(b.q_seed, b.q_len - w.k); b.t_seed[:] = np.minimum(b.t_seed, b.t_len - w.k)
ref = oracle.pairs(b.pool_u8, 0, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed, w.k, 1, -1, -1, 50, pool_len=b.pool_len)
db = logan.to_device(b)
for lvl in (None, 5, 6, 7):
    st = logan.new_stats()
    out, cells = logan.xdrop_batch(db, 1, -1, -1, 50, first_level=lvl, stats=st); torch.cuda.synchronize()
    o = out.cpu().numpy(); c = cells.cpu().numpy().view(np.uint64)
    bad = np.nonzero((o != ref[0]).any(axis=1) | (c != ref[1]))[0]
    print(lvl, "bad", len(bad), logan.stats_dict(st)["tasks_started"], [(int(p), o[p].tolist(), int(c[p]), ref[0][p].tolist(), int(ref[1][p])) for p in bad[:3]])
