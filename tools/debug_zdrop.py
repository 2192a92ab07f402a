import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_parity as T, datagen, oracle
import paper_2002_05200_b200 as logan
w = datagen.CONFIGS[1].with_(burst=0.5)
b = datagen.generate(w, n_pairs=120)
for Z in (0, 15):
    for X in (10, 200):
        ref = oracle.pairs_z(b.pool_u8, 0, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed, w.k, 1, -1, -1, X, Z, pool_len=b.pool_len)
        for lvl in (1, 2, 3, 4, 5, 6, 8):
            for lat in (False, True):
                for ho in (0, 40):
                    db = logan.to_device(b, 1)
                    st = logan.new_stats()
                    out, cells = logan.xdrop_batch(db, 1, -1, -1, X, first_level=lvl, latency_first=lat, handover=ho, zdrop=Z, stats=st)
                    torch.cuda.synchronize()
                    o = out.cpu().numpy(); c = cells.cpu().numpy().view(np.uint64)
                    bad = np.nonzero((o != ref[0]).any(axis=1) | (c != ref[1]))[0]
                    if len(bad):
                        print(f"Z={Z} X={X} lvl={lvl} lat={lat} ho={ho}: {len(bad)} bad", logan.stats_dict(st)["tasks_started"], flush=True)
print("done")
