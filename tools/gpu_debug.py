import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_parity as T
import paper_2002_05200_b200 as logan
b = T._mixed_pairs(7)
for X in (3, 10, 30):
    ref = T.oracle_run(b, X)
    for lvl in (1, 2, 3, 4, 5, 6):
        for lat in (False, True):
            for ho in (0, 2, 7):
                db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
                out, cells = logan.xdrop_batch(db, 1, -1, -1, X, first_level=lvl, latency_first=lat, handover=ho)
                torch.cuda.synchronize()
                o = out.cpu().numpy(); c = cells.cpu().numpy().view(np.uint64)
                bad = np.nonzero((o != ref[0]).any(axis=1) | (c != ref[1]))[0]
                sb = np.nonzero((o != ref[0]).any(axis=1))[0]
                print(f"X={X} lvl={lvl} lat={int(lat)} ho={ho}: bad={len(bad)} score-bad={len(sb)}", (o[bad[0]], c[bad[0]], ref[0][bad[0]], ref[1][bad[0]]) if len(bad) else "")
