"""Where the end-to-end (host-buffer) step loses against the device-timed one: the pool's
H2D copy alone, the host call on one stream (copies then sweep, serial) and on two streams
(bench.py's e2e: one step's copies overlap the previous sweep)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2002_05200_b200 as logan  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = datagen.CONFIGS[cfg]
if len(sys.argv) > 2:
    w = w.with_(xdrop=int(sys.argv[2]))
b = datagen.generate(w, n_pairs=w.n_pairs, u8=False)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
hp = [pin(x) for x in (b.pool_2bit, b.q_off, b.q_len, b.t_off, b.t_len, b.q_seed, b.t_seed)]
n = b.n_pairs
db = logan.to_device(b, logan.LOGAN_SEQ_2BIT)
K = int(os.environ.get("E2E_K", "10"))

def timed(fn, streams):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e0.record(streams[0])
    for s in streams[1:]:
        s.wait_event(e0)
    fn()
    ends = []
    for s in streams:
        e = torch.cuda.Event(enable_timing=True); e.record(s); ends.append(e)
    torch.cuda.synchronize()
    return max(e0.elapsed_time(e) for e in ends) / K

dpool = torch.empty(hp[0].numel(), dtype=torch.uint8, device="cuda")
s0, s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def h2d():
    with torch.cuda.stream(s0):
        for _ in range(K):
            dpool.copy_(hp[0], non_blocking=True)
print(f"pool {hp[0].numel()/1e6:.0f} MB: H2D {timed(h2d, [s0]):.2f} ms "
      f"({hp[0].numel() / 1e6 / timed(h2d, [s0]):.1f} GB/s)")
ws = logan.new_workspace(db) if hasattr(logan, "new_workspace") else None
out = torch.empty((n, 5), dtype=torch.int32, device="cuda"); cells = torch.empty(n, dtype=torch.int64, device="cuda")
def dev():
    for _ in range(K):
        logan.xdrop_batch(db, w.match, w.mismatch, w.gap, w.xdrop, out=out, cells=cells, stream=s0)
dev()  # warm-up (module loading, the per-stream workspace)
print(f"device-resident step (xdrop_batch, no workspace passed) {timed(dev, [s0]):.2f} ms")
arenas = [logan.HostArena(n, b.pool_len, logan.LOGAN_SEQ_2BIT, db.max_ext_len) for _ in range(3)]
hout = [torch.empty((n, 5), dtype=torch.int32).pin_memory().numpy() for _ in range(3)]
hcells = [torch.empty(n, dtype=torch.int64).pin_memory().numpy().view(np.uint64) for _ in range(3)]
hpn = [x.numpy() for x in hp]
def host(nstreams):
    streams = [s0, s1, s2][:nstreams]
    def run():
        for s in range(K):
            if s >= nstreams:
                streams[s % nstreams].synchronize()
            logan.xdrop_batch_host(hpn[0], logan.LOGAN_SEQ_2BIT, b.pool_len, *hpn[1:], w.k, w.match, w.mismatch,
                                   w.gap, w.xdrop, arenas[s % nstreams], out=hout[s % nstreams],
                                   cells=hcells[s % nstreams], stream=streams[s % nstreams], asynchronous=True)
    return run, streams
for ns in (1, 2, 3):
    run, streams = host(ns)
    run(); torch.cuda.synchronize()
    t0 = time.perf_counter(); ms = timed(run, streams); wall = (time.perf_counter() - t0) / K * 1e3
    print(f"host entry, {ns} stream(s): {ms:.2f} ms per step (host wall {wall:.2f})")

# the ideal pipelining: every sweep on ONE compute stream, each step's inputs copied on a
# separate copy stream (pinned -> device buffers) while the previous sweep runs
cs = torch.cuda.Stream()
NB = 2
dbs = [logan.to_device(b, logan.LOGAN_SEQ_2BIT) for _ in range(NB)]
hdev = [[hp[i] for i in range(7)] for _ in range(NB)]
free = [torch.cuda.Event() for _ in range(NB)]
done = [torch.cuda.Event() for _ in range(NB)]
def piped():
    for s in range(K):
        j = s % NB
        d = dbs[j]
        with torch.cuda.stream(cs):
            cs.wait_event(free[j])
            d.pool.copy_(hp[0], non_blocking=True)
            for dst, src in zip((d.q_off, d.q_len, d.t_off, d.t_len, d.q_seed, d.t_seed), hp[1:]):
                dst.copy_(src, non_blocking=True)
            done[j].record(cs)
        s0.wait_event(done[j])
        o, c = logan.xdrop_batch(d, w.match, w.mismatch, w.gap, w.xdrop, out=out, cells=cells, stream=s0)
        with torch.cuda.stream(s0):
            hout[j][:] = 0  # (host buffers unused here; results stay on the device)
        free[j].record(s0)
for e in free:
    e.record(s0)
piped(); torch.cuda.synchronize()
print(f"copy stream + one compute stream: {timed(piped, [s0, cs]):.2f} ms per step")

# the library's copy-ahead (options.flags bit 6): one stream, a ring of three arenas
es = torch.cuda.Stream()
done = [torch.cuda.Event() for _ in range(3)]
def ca_run():
    for s in range(K):
        if s >= 3:
            done[s % 3].synchronize()
        logan.xdrop_batch_host(hpn[0], logan.LOGAN_SEQ_2BIT, b.pool_len, *hpn[1:], w.k, w.match, w.mismatch,
                               w.gap, w.xdrop, arenas[s % 3], out=hout[s % 3], cells=hcells[s % 3], stream=es,
                               asynchronous=True, copy_ahead=True)
        done[s % 3].record(es)
ca_run(); torch.cuda.synchronize()
print(f"library copy-ahead, one stream, 3 arenas: {timed(ca_run, [es]):.2f} ms per step")
