"""e2e gap hunt: the library copy-ahead loop in a fresh process, then after a bench-like
device-timed section (timing events, L2 flush, stats run), then again."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2002_05200_b200 as logan  # noqa: E402

cfg, X = int(sys.argv[1]), int(sys.argv[2])
w = datagen.CONFIGS[cfg].with_(xdrop=X)
b = datagen.generate(w, n_pairs=w.n_pairs, u8=False)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
hp = [pin(x) for x in (b.pool_2bit, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed)]
n = b.n_pairs
db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
arenas = [logan.HostArena(n, b.pool_len, logan.LOGAN_SEQ_2BIT, db.max_ext_len) for _ in range(3)]
hout = [torch.empty((n, 5), dtype=torch.int32).pin_memory().numpy() for _ in range(3)]
hcells = [torch.empty(n, dtype=torch.int64).pin_memory().numpy().view(np.uint64) for _ in range(3)]
es = torch.cuda.Stream()
done = [torch.cuda.Event() for _ in range(3)]
K = 6

def ca(tag, first_level=None):
    def step(s):
        logan.xdrop_batch_host(hp[0], logan.LOGAN_SEQ_2BIT, b.pool_len, *hp[1:], w.k, w.match, w.mismatch,
                               w.gap, w.xdrop, arenas[s % 3], out=hout[s % 3], cells=hcells[s % 3], stream=es,
                               asynchronous=True, copy_ahead=True, first_level=first_level)
        done[s % 3].record(es)
    for s in range(3):
        step(s)
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(es)
    for s in range(K):
        if s >= 3:
            done[s % 3].synchronize()
        step(s)
    a1.record(es)
    torch.cuda.synchronize()
    print(f"{tag}: copy-ahead e2e {a0.elapsed_time(a1) / K:.2f} ms per step", flush=True)

ca("fresh")
# bench-like device-timed section
ws = logan.make_workspace(n, db.max_ext_len)
out = torch.empty((n, 5), dtype=torch.int32, device="cuda"); cells = torch.empty(n, dtype=torch.int64, device="cuda")
stream = torch.cuda.current_stream()
st = logan.new_stats()
logan.xdrop_batch(db, w.match, w.mismatch, w.gap, w.xdrop, workspace=ws, out=out, cells=cells, stats=st, stream=stream)
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
nst = logan._lib.N_STAGES
for s in range(5):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * nst)]
    for e in ev:
        e.record(stream)  # torch creates the CUDA event on its first record()
    flush.fill_(s & 0xff)
    logan.xdrop_batch(db, w.match, w.mismatch, w.gap, w.xdrop, workspace=ws, out=out, cells=cells,
                      stream=stream, timing_events=ev)
torch.cuda.synchronize()
ca("after a device-timed section")
ca("after, first_level=None again")
del flush
torch.cuda.synchronize()
ca("after freeing the flush buffer")
