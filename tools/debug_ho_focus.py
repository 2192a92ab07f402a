"""Repeat the hand-over-chain cases that failed nondeterministically (LOGAN_LIB picks the library)."""
import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_parity as T
import paper_2002_05200_b200 as logan
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 24
cases = [(140, 10, 2, False, 40), (140, 30, 6, False, 40), (102, 30, 6, False, 40), (106, 3, 5, True, 6),
         (102, 3, 1, True, 6)]
tot = 0
for seed, X, lvl, lat, ho in cases:
    b = T._mixed_pairs(seed)
    ref = T.oracle_run(b, X)
    nbad = 0
    for rep in range(reps):
        db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
        out, cells = logan.xdrop_batch(db, 1, -1, -1, X, first_level=lvl, latency_first=lat, handover=ho)
        torch.cuda.synchronize()
        o = out.cpu().numpy(); c = cells.cpu().numpy().view(np.uint64)
        bad = np.nonzero((o != ref[0]).any(axis=1) | (c != ref[1]))[0]
        nbad += bool(len(bad))
    tot += nbad
    print(os.environ.get("LOGAN_LIB", "main"), seed, X, lvl, lat, ho, f"{nbad}/{reps} bad", flush=True)
print("total bad", tot)
