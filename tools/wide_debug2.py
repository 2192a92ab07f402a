import sys
import numpy as np, torch
sys.path.insert(0, ".")
import datagen, oracle
import paper_2002_05200_b200 as logan
w = datagen.CONFIGS[4]
b = datagen.generate(w, n_pairs=6)
b.q_len[:] = np.minimum(b.q_len, 1200); b.t_len[:] = np.minimum(b.t_len, 1200)
b.q_seed[:] = np.minimum(b.q_seed, b.q_len - w.k); b.t_seed[:] = np.minimum(b.t_seed, b.t_len - w.k)
print("q_len", b.q_len, "q_seed", b.q_seed, "t_len", b.t_len, "t_seed", b.t_seed, "maxext", b.max_ext_len())
ref = oracle.pairs(b.pool_u8, 0, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed, w.k, 1, -1, -1, 50, pool_len=b.pool_len)
print("oracle cells", int(ref[1].sum()), ref[1].tolist())
db = logan.to_device(b)
for lvl in (None, 6, 7):
    out, cells = logan.xdrop_batch(db, 1, -1, -1, 50, first_level=lvl); torch.cuda.synchronize()
    o = out.cpu().numpy(); c = cells.cpu().numpy().view(np.uint64)
    print(lvl, int(c.sum()), c.tolist(), [(p, o[p].tolist(), ref[0][p].tolist()) for p in range(len(c)) if (o[p] != ref[0][p]).any()])
