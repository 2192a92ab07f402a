#!/usr/bin/env python
"""Benchmark of the B200 X-drop hot path (LOGAN, arXiv 2002.05200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the whole hot path (task expansion + LPT bucketing +
all sweep levels + combine) over one batch of synthetic pairs already resident
in HBM.  Default workload: BASELINE.json configs[1] = 100K pairs of 2.5 kb
reads, 15% error, k = 17, X = 20, +1/-1/-1 (``datagen.CONFIGS[2]``); under
torchrun every rank processes its own 100K pairs (weak scaling, no data-path
collective; results are gathered once after the timed region).

Metric: GCUPS = band cells (the oracle's definition, c-amb-14) / device time,
aggregated over all ranks with the max-over-ranks time.  Prints ONE JSON line
on rank 0.  DESIGN.md §7 documents every key.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "GCUPS (computed cells/s, device-timed) at 1/2/4/8 B200 vs int roofline"
UNIT = "GCUPS"
N_REF_OPS_PER_CELL = 6       # algorithmic int32 ops per cell (SURVEY §8d convention)
ALU_LANES_PER_SM_CLK = 64    # 4 SMSPs x 16 int32 ALU lanes (B300_MICROARCH: alu pipe rt_SMSP = 2)
B200_SMS = 148


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2,
                    help="datagen.CONFIGS key (BASELINE configs[c-1]); 7 = protein-like pairs scored with a "
                         "substitution matrix (SURVEY §8f row 4)")
    ap.add_argument("--pairs", type=int, default=None, help="pairs per GPU (default: the config's)")
    ap.add_argument("--xdrop", type=int, default=None)
    ap.add_argument("--zdrop", type=int, default=None,
                    help="also stop extensions by Z-drop with this Z (DESIGN.md c-amb-19; off by default)")
    ap.add_argument("--fmt", choices=["2bit", "u8"], default="2bit")
    ap.add_argument("--first-level", type=int, default=0)
    ap.add_argument("--latency-first", action="store_true",
                    help="run the first level in its latency shape (one warp per task)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target host seconds of the oracle sample (cpu_baseline)")
    ap.add_argument("--ref-step-seconds", type=float, default=2.0,
                    help="target host seconds per step of --impl reference")
    ap.add_argument("--stats", action="store_true", help="print per-level stats to stderr")
    return ap.parse_args()


PROTEIN_CONFIG = 7  # not a BASELINE config: SURVEY §8f row 4 (substitution matrices)
PROTEIN_PAIRS = 100_000


def workload(args):
    import datagen
    if args.config == PROTEIN_CONFIG:
        n = args.pairs if args.pairs is not None else PROTEIN_PAIRS
        w = datagen.protein_pairs(0, xdrop=args.xdrop if args.xdrop is not None else 50).workload
        return w, n
    w = datagen.CONFIGS[args.config]
    if args.xdrop is not None:
        w = w.with_(xdrop=args.xdrop)
    n = args.pairs if args.pairs is not None else w.n_pairs
    return w, n


def make_batch(args, w, n, pair_base=0, u8=False, two_bit=True):
    import datagen
    if args.config == PROTEIN_CONFIG:
        return datagen.protein_pairs(n, pair_base=pair_base, xdrop=w.xdrop, gap=w.gap)
    return datagen.generate(w, n_pairs=n, pair_base=pair_base, u8=u8, two_bit=two_bit)


ZDROP = None  # set from --zdrop in main / run_reference


def run_oracle(batch, w, sl, threads):
    """The oracle on pairs ``sl`` of the batch -> per-pair cells."""
    import oracle
    import datagen
    if ZDROP is not None:
        sub = datagen.protein_matrix() if batch.pool_2bit is None else None
        pool, fmt = (batch.pool_u8, 0) if sub is not None else (batch.pool_2bit, 1)
        _, cells = oracle.pairs_z(pool, fmt, batch.q_off[sl], batch.q_len[sl], batch.t_off[sl], batch.t_len[sl],
                                  batch.q_seed[sl], batch.t_seed[sl], w.k, w.match, w.mismatch, w.gap, w.xdrop,
                                  ZDROP, subst=sub, pool_len=batch.pool_len, n_threads=threads)
        return cells
    if batch.pool_2bit is None:  # protein codes: the substitution-matrix oracle
        _, cells = oracle.pairs_subst(batch.pool_u8, batch.q_off[sl], batch.q_len[sl], batch.t_off[sl],
                                      batch.t_len[sl], batch.q_seed[sl], batch.t_seed[sl], w.k,
                                      datagen.protein_matrix(), w.gap, w.xdrop, pool_len=batch.pool_len,
                                      n_threads=threads)
        return cells
    _, cells = oracle.pairs(batch.pool_2bit, 1, batch.q_off[sl], batch.q_len[sl], batch.t_off[sl],
                            batch.t_len[sl], batch.q_seed[sl], batch.t_seed[sl], w.k, w.match,
                            w.mismatch, w.gap, w.xdrop, pool_len=batch.pool_len, n_threads=threads)
    return cells


def config_dict(w, n, fmt, first_level, world):
    d = {"workload": w.name, "pairs_per_gpu": n, "total_pairs": n * world,
         "read_len": (f"{w.tlen_min}-{w.tlen_max} residues" if w.name.startswith("protein") else
                      w.tlen_max if w.mode == 0 else f"{w.len_lo}-{w.len_hi}"),
         "error": w.err, "k": w.k, "X": w.xdrop,
         "scoring": (f"synthetic 20x20 substitution matrix (datagen.protein_matrix), gap {w.gap:+d}"
                     if w.name.startswith("protein") else f"{w.match:+d}/{w.mismatch:+d}/{w.gap:+d}"),
         "fmt": fmt,
         "seed": w.seed, "l2": "flushed between timed steps (256 MiB write)",
         "parallelism": f"pairs sharded over {world} GPU(s), no data-path collective"}
    if first_level:
        d["first_level"] = first_level
    if ZDROP is not None:
        d["zdrop"] = ZDROP
    return d


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device_uuid: str | None):
        self.uuid = device_uuid
        self.proc = None

    def start(self):
        cmd = ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50"]
        if self.uuid:
            cmd += ["-i", self.uuid]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], None, set()
        for line in out.splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- oracle legs
def oracle_sample(batch, w, seconds, threads):
    """Time the oracle as it stands on a bounded prefix of the batch."""
    import numpy as np
    import oracle
    oracle.build()

    def run(k):
        sl = slice(0, k)
        t0 = time.perf_counter()
        cells = run_oracle(batch, w, sl, threads)
        return time.perf_counter() - t0, int(np.asarray(cells, dtype=np.uint64).sum())

    k = min(batch.n_pairs, max(threads * 4, 64))
    dt, cells = run(k)
    if dt < seconds * 0.5 and k < batch.n_pairs:
        k = min(batch.n_pairs, max(k + 1, int(k * seconds / max(dt, 1e-3))))
        dt, cells = run(k)
    return {"pairs": k, "seconds": dt, "cells": cells}


def run_reference(args):
    """--impl reference: the oracle (the only reference this tier has) on host cores."""
    global ZDROP
    ZDROP = args.zdrop
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import datagen
    w, n = workload(args)
    threads = len(os.sched_getaffinity(0))
    probe = make_batch(args, w, min(n, max(threads * 1024, 4096)))
    cal = oracle_sample(probe, w, args.ref_step_seconds, threads)
    per_step = cal["pairs"]
    batch = make_batch(args, w, min(n, per_step))
    times, cells = [], 0
    for s in range(args.warmup + args.steps):
        import numpy as np
        t0 = time.perf_counter()
        c = run_oracle(batch, w, slice(0, batch.n_pairs), threads)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            cells = int(np.asarray(c, dtype=np.uint64).sum())
    total = sum(times)
    value = cells * len(times) / total / 1e9
    sample = (f"first {batch.n_pairs} of the {n} pairs of {w.name} per step "
              f"({cells} cells/step), oracle_pairs on {threads} host threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": config_dict(w, n, "u8" if args.config == PROTEIN_CONFIG else "2bit", 0, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- our arm
def main():
    global ZDROP
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    ZDROP = args.zdrop

    import numpy as np
    import torch
    import torch.distributed as dist

    import datagen
    from paper_2002_05200_b200 import build as _build
    _build.build()
    import paper_2002_05200_b200 as logan

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    w, n = workload(args)
    protein = args.config == PROTEIN_CONFIG
    if protein:
        args.fmt = "u8"
    fmt = logan.LOGAN_SEQ_2BIT if args.fmt == "2bit" else logan.LOGAN_SEQ_U8
    batch = make_batch(args, w, n, pair_base=rank * n, u8=(args.fmt == "u8"), two_bit=True)
    subst = torch.as_tensor(datagen.protein_matrix()).to(dev) if protein else None
    db = logan.to_device(batch, fmt, device=dev)
    ws = logan.make_workspace(n, db.max_ext_len, dev)
    out = torch.empty((n, 5), dtype=torch.int32, device=dev)
    cells = torch.empty(n, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    first = args.first_level or None

    def step(events=None, stats=None):
        logan.xdrop_batch(db, w.match, w.mismatch, w.gap, w.xdrop, workspace=ws, out=out, cells=cells,
                          stats=stats, first_level=first, stream=stream, timing_events=events,
                          latency_first=args.latency_first, subst=subst, zdrop=args.zdrop)

    # one untimed run with device stats: per-level task and cell counts (deterministic)
    st = logan.new_stats(dev)
    step(stats=st)
    torch.cuda.synchronize()
    stats = logan.stats_dict(st)
    cells_step = int(cells.sum().item())
    assert cells_step == stats["cells_total"], (cells_step, stats["cells_total"])
    if args.stats and rank == 0:
        print(json.dumps(stats), file=sys.stderr)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    nst = logan._lib.N_STAGES
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * nst)] for _ in range(args.steps)]
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for e in [x for row in ev for x in row] + e0 + e1:
        e.record(stream)  # torch creates the CUDA event lazily on its first record()
    torch.cuda.synchronize()
    props = torch.cuda.get_device_properties(dev)
    uuid = getattr(props, "uuid", None)
    sampler = ClockSampler(f"GPU-{uuid}" if uuid is not None and not str(uuid).startswith("GPU-") else
                           (str(uuid) if uuid is not None else None))
    if world > 1:
        dist.barrier(device_ids=[local])
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.1)
    for s in range(args.steps):
        flush.fill_(s & 0xff)
        e0[s].record(stream)
        step(events=ev[s])
        e1[s].record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if world > 1:
        dist.barrier(device_ids=[local])
    step_ms = [e0[s].elapsed_time(e1[s]) for s in range(args.steps)]
    total_ms = sum(step_ms)

    # per-stage device times (events recorded by the library on this stream)
    stage_ms = {}
    for stg in range(nst):
        try:
            stage_ms[stg] = sum(ev[s][2 * stg].elapsed_time(ev[s][2 * stg + 1]) for s in range(args.steps))
        except RuntimeError:
            pass  # stage not launched in this configuration
    n_launch_stages = [stg for stg in stage_ms if 1 <= stg <= nst - 2]
    launches_per_step = 3 + len(n_launch_stages) + 1  # expand, scan, scatter, levels, combine

    # max over ranks (time), sum over ranks (cells)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    c = torch.tensor([cells_step], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
    total_ms_max = float(t.item())
    cells_all = int(c.item())
    value = cells_all * args.steps / (total_ms_max / 1e3) / 1e9

    # gather of per-pair results to rank 0 (outside the timed steps, reported separately)
    gather_ms = None
    if world > 1:
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        res = torch.cat([out.view(torch.int32), cells.view(torch.int32).view(n, 2)], dim=1).contiguous()
        allres = torch.empty((world * n, 7), dtype=torch.int32, device=dev)
        g0.record(stream)
        dist.all_gather_into_tensor(allres, res)
        g1.record(stream)
        torch.cuda.synchronize()
        gather_ms = g0.elapsed_time(g1)

    # dominant kernel and its roofline (bound: int32 ALU)
    dom_stage = max((s for s in stage_ms if 1 <= s <= nst - 2), key=lambda s: stage_ms[s])
    dom_level = dom_stage - 1
    dom_ms = stage_ms[dom_stage] / args.steps
    dom_cells = stats["cells_per_level"][dom_level]
    sm_max = clocks.get("sm_max_mhz") or 1965.0
    peak_tops = B200_SMS * ALU_LANES_PER_SM_CLK * sm_max * 1e6 / 1e12
    achieved_tops = N_REF_OPS_PER_CELL * dom_cells / (dom_ms / 1e3) / 1e12
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            tj = json.load(open(tfile))
            key = f"{w.name}/{args.fmt}/level{dom_level + 1}"
            traffic = tj.get(key)
        except (OSError, ValueError):
            traffic = None
    # the library picks window widths from X (from ceil(X / |gap|) with a substitution matrix)
    xband = -(-w.xdrop // -w.gap) if subst is not None else w.xdrop
    level_names = [f"window{logan._lib.load().logan_level_width(lv + 1, xband, db.max_ext_len, 0)}"
                   for lv in range(6)] + ["band8192", "wide_cta"]
    roofline = {"bound": "alu", "achieved": achieved_tops, "peak": peak_tops, "unit": "TOP/s",
                "frac": achieved_tops / peak_tops, "traffic": traffic,
                "kernel": f"{'k_window' if dom_level < 6 else ('k_band' if dom_level == 6 else 'k_wide')} "
                          f"level {dom_level + 1} ({level_names[dom_level]})",
                "kernel_ms": dom_ms, "kernel_share_of_step": dom_ms / (total_ms / args.steps),
                "ops_per_cell": N_REF_OPS_PER_CELL,
                "peak_derivation": f"{B200_SMS} SMs x {ALU_LANES_PER_SM_CLK} int32 lanes/clk x {sm_max:.0f} MHz"}

    # End-to-end through the host-buffer C-ABI entry point, from pinned host memory:
    # every step copies its inputs in (H2D) and its results out (D2H) inside the timed
    # region. Steps alternate between two arenas / streams (logan_xdrop_batch_host_async),
    # so one step's copies overlap the previous step's sweep.
    e2e = None
    if not args.no_e2e:
        pool_np = batch.pool_2bit if fmt == logan.LOGAN_SEQ_2BIT else batch.pool_u8
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        hp = [pin(x) for x in (pool_np, batch.q_off, batch.q_len, batch.t_off, batch.t_len,
                               batch.q_seed, batch.t_seed)]
        hout = [torch.empty((n, 5), dtype=torch.int32).pin_memory().numpy() for _ in range(2)]
        hcells = [torch.empty(n, dtype=torch.int64).pin_memory().numpy().view(np.uint64) for _ in range(2)]
        arenas = [logan.HostArena(n, batch.pool_len, fmt, db.max_ext_len, device=dev) for _ in range(2)]
        streams = [torch.cuda.Stream(dev) for _ in range(2)]
        pool_bytes = (batch.pool_len + 3) // 4 if fmt == logan.LOGAN_SEQ_2BIT else batch.pool_len

        def e2e_step(s):
            logan.xdrop_batch_host(hp[0], fmt, batch.pool_len, *hp[1:], w.k, w.match, w.mismatch,
                                   w.gap, w.xdrop, arenas[s % 2], out=hout[s % 2], cells=hcells[s % 2],
                                   first_level=first, stream=streams[s % 2], asynchronous=True, subst=subst,
                                   zdrop=args.zdrop)

        for s_ in range(2):
            e2e_step(s_)
        torch.cuda.synchronize()
        ke = max(4, args.steps)  # same K as the device-timed steps (steady state)
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a0.record(streams[0])
        streams[1].wait_event(a0)
        for s_ in range(ke):
            if s_ >= 2:
                streams[s_ % 2].synchronize()  # step s-2's outputs are read before its buffers are reused
                assert int(hcells[s_ % 2].sum()) == cells_step
            e2e_step(s_)
        ends = []
        for st_ in streams:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(st_)
            ends.append(ev)
        torch.cuda.synchronize()
        e2e_ms = max(a0.elapsed_time(ev) for ev in ends)
        te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        for hc in hcells:
            assert int(hc.sum()) == cells_step
        e2e = {"value": cells_all * ke / (float(te.item()) / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(pool_bytes + 32 * n), "d2h_bytes_per_step": int(28 * n),
               "steps": ke, "api": "logan_xdrop_batch_host_async (2 arenas / 2 streams, pinned)"}

    # CPU baseline: the oracle on this host's cores, rank 0 at N = 1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        r = oracle_sample(batch, w, args.cpu_seconds, threads)
        cpu = {"value": r["cells"] / r["seconds"] / 1e9, "unit": UNIT, "cores": threads,
               "kind": "oracle",
               "sample": f"first {r['pairs']} of the {n} pairs ({r['cells']} cells) in "
                         f"{r['seconds']:.1f} s, oracle_pairs on {threads} host threads"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
                "data": "synthetic (datagen, seeded; DESIGN.md §5)",
                "config": config_dict(w, n, args.fmt, args.first_level, world),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_per_step * args.steps, "clocks": clocks,
                "cells_per_step": cells_all,
                "stage_ms_per_step": {str(k): v / args.steps for k, v in stage_ms.items()},
                "levels": {"tasks_started": stats["tasks_started"],
                           "tasks_finished": stats["tasks_finished"],
                           "cells_per_level": stats["cells_per_level"],
                           "window_shifts": stats["window_shifts"]}}
        if gather_ms is not None:
            line["gather_ms"] = gather_ms
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
