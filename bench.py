#!/usr/bin/env python
"""Benchmark of the B200 X-drop hot path (LOGAN, arXiv 2002.05200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C] [--xdrop X] [--share r/N]

One step = one pass of the whole hot path (task expansion + LPT bucketing +
all sweep levels + combine) over one batch of synthetic pairs already resident
in HBM.  Default workload: BASELINE.json configs[2] = 100K pairs of 10 kb reads,
15% error, k = 17, X = 20, +1/-1/-1 (``datagen.CONFIGS[3]``), the config the
metric is quoted on "at 1/2/4/8 B200"; ``--config 2`` is configs[1] (2.5 kb).

Multi-GPU (torchrun, N ranks): the config's ONE batch is split across the
ranks by a static cell-count-balanced LPT partition (paper P:223-225,
``multi.partition_lpt`` over ``multi.pair_costs``) -- strong scaling, no
collective on the data path; after the timed region the per-pair results are
gathered once to rank 0 and compared with a 1-GPU run of the whole batch.
``--share r/N`` runs rank r's share of an N-way split on one GPU (per-share
times project the N-GPU makespan without an N-GPU box).

Metric: GCUPS = band cells (the oracle's definition, c-amb-14) / device time,
aggregated over all ranks with the max-over-ranks time.  The timed output is
checked element by element against the oracle on a sample ("parity"); any
mismatch exits non-zero.  Prints ONE JSON line on rank 0.
documents every key.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
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
B200_SMS = 148
DEFAULT_CONFIG = 3
PEAK_FILE = os.path.join(ROOT, "profiles", "int_peak.json")      # tools/int_peak.py (microbenchmark)
NCU_FILE = os.path.join(ROOT, "profiles", "ncu_metrics.json")    # tools/ncu_metrics.py (ncu --set full)


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG,
                    help="datagen.CONFIGS key (BASELINE configs[c-1]); 7 = protein-like pairs scored with a "
                         "substitution matrix (SURVEY §8f row 4)")
    ap.add_argument("--pairs", type=int, default=None, help="pairs of the whole batch (default: the config's)")
    ap.add_argument("--xdrop", type=int, default=None)
    ap.add_argument("--zdrop", type=int, default=None,
                    help="also stop extensions by Z-drop with this Z (DESIGN.md c-amb-19; off by default)")
    ap.add_argument("--fmt", choices=["2bit", "u8"], default="2bit")
    ap.add_argument("--no-pack-u8", action="store_true",
                    help="--fmt u8: run the u8 kernels (default: logan_pack_2bit re-encodes an A/C/G/T pool "
                         "on the device every step, then the 2-bit path)")
    ap.add_argument("--first-level", type=int, default=0)
    ap.add_argument("--first-slots", type=int, default=0,
                    help="tuning knob: force the first window's slots (16/20/24/28/32; 0 = automatic)")
    ap.add_argument("--latency-first", action="store_true",
                    help="run the first level in its latency shape (one warp per task)")
    ap.add_argument("--throughput-first", action="store_true",
                    help="tuning knob: run the first level in its throughput shape even with few tasks")
    ap.add_argument("--share", default=None,
                    help="r/N: run only rank r's share of an N-way split of the batch, on one GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="N > 1: skip the gathered-vs-1-GPU check")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target host seconds of the oracle sample (cpu_baseline)")
    ap.add_argument("--parity-seconds", type=float, default=4.0,
                    help="target host seconds of the oracle parity sample when cpu_baseline does not run")
    ap.add_argument("--ref-step-seconds", type=float, default=2.0,
                    help="target host seconds per step of --impl reference")
    ap.add_argument("--stats", action="store_true", help="print per-level stats to stderr")
    return ap.parse_args(argv)


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


def shard_of(args, w, n, world, rank):
    """Global pair indices of rank ``rank``'s share of the n-pair batch (all of
    it at world 1) and the partition (None at world 1)."""
    import numpy as np
    if world == 1:
        return np.arange(n, dtype=np.int64), None
    if args.config == PROTEIN_CONFIG:  # no length pass for the numpy protein generator: even ranges
        bounds = [n * r // world for r in range(world + 1)]
        parts = [np.arange(bounds[r], bounds[r + 1], dtype=np.int64) for r in range(world)]
        return parts[rank], parts
    import datagen
    from paper_2002_05200_b200 import multi
    ql, tl, qs, ts = datagen.lengths(w, n)
    parts = multi.partition_lpt(multi.pair_costs(ql, tl, qs, ts, w.k, w.xdrop, w.gap), world)
    return parts[rank], parts


def make_batch(args, w, idx, u8=False):
    """The pairs ``idx`` (global indices, ascending) of the workload."""
    import datagen
    n = len(idx)
    if args.config == PROTEIN_CONFIG:
        base = int(idx[0]) if n else 0
        return datagen.protein_pairs(n, pair_base=base, xdrop=w.xdrop, gap=w.gap)
    if n and int(idx[-1]) - int(idx[0]) + 1 == n:  # a contiguous range
        return datagen.generate(w, n_pairs=n, pair_base=int(idx[0]), u8=u8, two_bit=True)
    return datagen.generate(w, indices=idx, u8=u8, two_bit=True)


ZDROP = None  # set from --zdrop in main / run_reference


def run_oracle(batch, w, sl, threads):
    """The oracle on pairs ``sl`` of the batch -> (int32[n,5] results, uint64[n] cells)."""
    import oracle
    import datagen
    if ZDROP is not None:
        sub = datagen.protein_matrix() if batch.pool_2bit is None else None
        pool, fmt = (batch.pool_u8, 0) if sub is not None else (batch.pool_2bit, 1)
        return oracle.pairs_z(pool, fmt, batch.q_off[sl], batch.q_len[sl], batch.t_off[sl], batch.t_len[sl],
                              batch.q_seed[sl], batch.t_seed[sl], w.k, w.match, w.mismatch, w.gap, w.xdrop,
                              ZDROP, subst=sub, pool_len=batch.pool_len, n_threads=threads)
    if batch.pool_2bit is None:  # protein codes: the substitution-matrix oracle
        return oracle.pairs_subst(batch.pool_u8, batch.q_off[sl], batch.q_len[sl], batch.t_off[sl],
                                  batch.t_len[sl], batch.q_seed[sl], batch.t_seed[sl], w.k,
                                  datagen.protein_matrix(), w.gap, w.xdrop, pool_len=batch.pool_len,
                                  n_threads=threads)
    return oracle.pairs(batch.pool_2bit, 1, batch.q_off[sl], batch.q_len[sl], batch.t_off[sl],
                        batch.t_len[sl], batch.q_seed[sl], batch.t_seed[sl], w.k, w.match,
                        w.mismatch, w.gap, w.xdrop, pool_len=batch.pool_len, n_threads=threads)


def config_dict(w, n, fmt, first_level, world, share=None):
    d = {"workload": w.name, "total_pairs": n,
         "read_len": (f"{w.tlen_min}-{w.tlen_max} residues" if w.name.startswith("protein") else
                      w.tlen_max if w.mode == 0 else f"{w.len_lo}-{w.len_hi}"),
         "error": w.err, "k": w.k, "X": w.xdrop,
         "scoring": (f"synthetic 20x20 substitution matrix (datagen.protein_matrix), gap {w.gap:+d}"
                     if w.name.startswith("protein") else f"{w.match:+d}/{w.mismatch:+d}/{w.gap:+d}"),
         "fmt": fmt,
         "seed": w.seed, "l2": "flushed between timed steps (256 MiB write)",
         "parallelism": (f"one batch split over {world} GPU(s) by a static cell-count-balanced LPT partition "
                         "(multi.pair_costs); no data-path collective, one gather after the timed region")}
    if share is not None:
        d["share"] = f"{share[0]}/{share[1]}"
        d["parallelism"] = (f"share {share[0]} of a {share[1]}-way LPT split of the batch, run alone on one GPU "
                            "(projects the per-GPU time of an N-GPU run)")
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
def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.TimeoutExpired):
        pass
    return platform.processor() or "unknown"


def oracle_sample(batch, w, seconds, threads, idx_pool=None):
    """Time the oracle as it stands on a bounded sample of the batch: pairs
    ``idx_pool[:k]`` (default: the batch order), k grown to about ``seconds``."""
    import numpy as np
    import oracle
    oracle.build()
    if idx_pool is None:
        idx_pool = np.arange(batch.n_pairs)

    def run(k):
        sl = idx_pool[:k]
        t0 = time.perf_counter()
        o, c = run_oracle(batch, w, sl, threads)
        return time.perf_counter() - t0, o, c

    k = min(len(idx_pool), max(threads * 4, 64))
    dt, o, c = run(k)
    if dt < seconds * 0.5 and k < len(idx_pool):
        k = min(len(idx_pool), max(k + 1, int(k * seconds / max(dt, 1e-3))))
        dt, o, c = run(k)
    return {"idx": idx_pool[:k], "seconds": dt, "out": o, "cells": c,
            "cell_sum": int(np.asarray(c, dtype=np.uint64).sum())}


def single_thread_c1():
    """The oracle on BASELINE configs[0] (C1, 1,000 pairs) on ONE host thread."""
    import datagen
    import numpy as np
    w = datagen.CONFIGS[1]
    b = datagen.generate(w, u8=False)
    t0 = time.perf_counter()
    _, c = run_oracle(b, w, slice(0, b.n_pairs), 1)
    dt = time.perf_counter() - t0
    return {"value": int(np.asarray(c, np.uint64).sum()) / dt / 1e9, "unit": UNIT,
            "workload": f"{w.name} ({b.n_pairs} pairs, 1 thread, {dt:.2f} s)"}


def run_reference(args):
    """--impl reference: the oracle (the only reference this tier has) on host cores."""
    global ZDROP
    ZDROP = args.zdrop
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    w, n = workload(args)
    threads = len(os.sched_getaffinity(0))
    probe = make_batch(args, w, np.arange(min(n, max(threads * 1024, 4096))))
    cal = oracle_sample(probe, w, args.ref_step_seconds, threads)
    per_step = len(cal["idx"])
    batch = make_batch(args, w, np.arange(min(n, per_step)))
    times, cells = [], 0
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        _, c = run_oracle(batch, w, slice(0, batch.n_pairs), threads)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            cells = int(np.asarray(c, dtype=np.uint64).sum())
    total = sum(times)
    value = cells * len(times) / total / 1e9
    sample = (f"first {batch.n_pairs} of the {n} pairs of {w.name} per step "
              f"({cells} cells/step), oracle_pairs on {threads} host threads ({cpu_model()})")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": config_dict(w, n, "u8" if args.config == PROTEIN_CONFIG else "2bit", 0, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- roofline inputs
def int_peak(sm_max_mhz, packed):
    """Peak ALU-pipe integer ops/s of the B200: the measured per-SM per-clock
    throughput of the cell's ALU-pipe instructions (tools/int_peak.py,
    profiles/int_peak.json) x 148 SMs x the max SM clock -- for a kernel whose
    cells run on packed .S16x2 DPX instructions (two lanes per instruction) the
    16x2 peak ("must be stated with the 16x2 peak"), else the int32
    one. Without the file, the guide's ALU pipe rate (16 lanes per SMSP, 64 per
    SM; doubled for 16x2). Returns (peak TOP/s, derivation, int32 peak TOP/s)."""
    try:
        pk = json.load(open(PEAK_FILE))
        l32 = float(pk["alu_int32_ops_per_clk_per_sm"])
        l16 = float(pk["s16x2_ops_per_clk_per_sm"])
        src = f"measured: {pk.get('source', PEAK_FILE)}"
    except (OSError, ValueError, KeyError):
        l32, l16 = 64.0, 128.0
        src = "derived: 4 SMSPs x 16-lane ALU pipe"
    lanes = l16 if packed else l32
    how = (f"{B200_SMS} SMs x {lanes:.1f} {'16x2 lane-ops' if packed else 'int32 ops'}/clk/SM on the ALU pipe "
           f"({src}) x {sm_max_mhz:.0f} MHz")
    f = B200_SMS * sm_max_mhz * 1e6 / 1e12
    return lanes * f, how, l32 * f


def ncu_evidence(key):
    """Per-launch ncu counters of the dominant kernel for this workload (committed
    under profiles/ by tools/ncu_metrics.py from an `ncu --set full` capture)."""
    try:
        return json.load(open(NCU_FILE)).get(key)
    except (OSError, ValueError):
        return None


# --------------------------------------------------------------------------- our arm
def main(argv=None):
    global ZDROP
    args = parse_args(argv)
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
    share = None
    if args.share:
        if world > 1:
            raise SystemExit("--share runs one share on one GPU (no torchrun)")
        r, nsh = (int(x) for x in args.share.split("/"))
        share = (r, nsh)

    w, n = workload(args)
    protein = args.config == PROTEIN_CONFIG
    if protein:
        args.fmt = "u8"
    fmt = logan.LOGAN_SEQ_2BIT if args.fmt == "2bit" else logan.LOGAN_SEQ_U8
    if share is not None:
        idx, parts = shard_of(args, w, n, share[1], share[0])
    else:
        idx, parts = shard_of(args, w, n, world, rank)
    batch = make_batch(args, w, idx, u8=(args.fmt == "u8"))
    n_local = batch.n_pairs
    subst = torch.as_tensor(datagen.protein_matrix()).to(dev) if protein else None
    db = logan.to_device(batch, fmt, device=dev)
    ws = logan.make_workspace(n_local, db.max_ext_len, dev)
    out = torch.empty((n_local, 5), dtype=torch.int32, device=dev)
    cells = torch.empty(n_local, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    first = args.first_level or None

    pack_u8 = fmt == logan.LOGAN_SEQ_U8 and subst is None and not args.no_pack_u8
    u8_packed = False
    if pack_u8:  # does the pool take the packed path (all bytes A/C/G/T)?
        u8_packed = int(logan.pack_2bit(db, stream)[1].item()) == 0

    def step(events=None, stats=None):
        logan.xdrop_batch(db, w.match, w.mismatch, w.gap, w.xdrop, workspace=ws, out=out, cells=cells,
                          stats=stats, first_level=first, stream=stream, timing_events=events,
                          latency_first=args.latency_first, subst=subst, zdrop=args.zdrop, pack_u8=pack_u8,
                          first_slots=args.first_slots, throughput_first=args.throughput_first)

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
    # [pack,] expand, scan, scatter, the levels, combine: the first level is one launch, a
    # later window level two (latency and throughput shapes, one exits at once), the band
    # level two (its two stages), the CTA level one
    first_stage = stats["first_level"]  # stage of the first level (stage s = level s)
    per_stage = lambda stg: 1 if (stg == first_stage or stg == nst - 2) else 2
    launches_per_step = 3 + sum(per_stage(stg) for stg in n_launch_stages) + 1 + int(pack_u8)

    # max over ranks (time), sum over ranks (cells)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    c = torch.tensor([cells_step], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
    total_ms_max = float(t.item())
    cells_all = int(c.item())
    value = cells_all * args.steps / (total_ms_max / 1e3) / 1e9
    out_h = out.cpu().numpy()
    cells_h = cells.cpu().numpy().view(np.uint64)

    # dominant kernel and its roofline (bound: int32 ALU)
    dom_stage = max((s for s in stage_ms if 1 <= s <= nst - 2), key=lambda s: stage_ms[s])
    dom_level = dom_stage - 1
    dom_ms = stage_ms[dom_stage] / args.steps
    dom_cells = stats["cells_per_level"][dom_level]
    sm_max = clocks.get("sm_max_mhz") or 1965.0
    # the packed int16 kernels: the register windows of a 2-bit pool at X <= 16000 (no
    # Z-drop, no matrix; options.flags bit 4 off) except the int32 one-warp shapes of
    # W <= 64, and the band level
    first_lv = stats.get("first_level", 0) - 1  # (not `first`: that is the e2e calls' first_level)
    lat_narrow = (dom_level == first_lv and stats.get("first_shape") == "latency"
                  and 0 < stats.get("first_width", 0) <= 64)
    # (a Z >= X' never fires: the library then runs the plain, packed build)
    zdrop_on = args.zdrop is not None and args.zdrop < w.xdrop
    packed = (dom_level <= 5 and (fmt == logan.LOGAN_SEQ_2BIT or u8_packed) and w.xdrop <= 16000
              and not zdrop_on and not protein and not lat_narrow) or dom_level == 6
    peak_tops, peak_how, peak32 = int_peak(sm_max, packed)
    achieved_tops = N_REF_OPS_PER_CELL * dom_cells / (dom_ms / 1e3) / 1e12
    # the library picks window widths from X (from ceil(X / |gap|) with a substitution matrix)
    xband = -(-w.xdrop // -w.gap) if subst is not None else w.xdrop
    level_names = [f"window{logan._lib.load().logan_level_width(lv + 1, xband, db.max_ext_len, 0)}"
                   for lv in range(6)] + ["band, 4096 / 8192-slot rings", "wide_cta"]
    ncu_key = f"{w.name}/{args.fmt}/level{dom_level + 1}"
    ev_ncu = ncu_evidence(ncu_key)
    roofline = {"bound": "alu", "achieved": achieved_tops, "peak": peak_tops, "unit": "TOP/s",
                "frac": achieved_tops / peak_tops,
                "traffic": ev_ncu.get("dram_bytes") if ev_ncu else None,
                "kernel": f"{'k_window' if dom_level < 6 else ('k_band' if dom_level == 6 else 'k_wide')} "
                          f"level {dom_level + 1} ({level_names[dom_level]})",
                "kernel_ms": dom_ms, "kernel_share_of_step": dom_ms / (total_ms / args.steps),
                "ops_per_cell": N_REF_OPS_PER_CELL, "cells_per_launch": dom_cells,
                "peak_derivation": peak_how, "packed_16x2": packed,
                "frac_vs_int32_alu_peak": achieved_tops / peak32}
    if ev_ncu:
        roofline["ncu"] = {k: ev_ncu[k] for k in ("sass_thread_inst_per_cell", "int_thread_inst_per_cell",
                                                  "int_warp_gips", "alu_pipe_pct", "fma_pipe_pct", "issue_pct",
                                                  "source") if k in ev_ncu}

    # End-to-end through the host-buffer C-ABI entry point, from pinned host memory:
    # every step copies its inputs in (H2D) and its results out (D2H) inside the timed
    # region (logan_xdrop_batch_host_async, one stream, a ring of arenas, copy-ahead).
    e2e = None
    if not args.no_e2e:
        pool_np = batch.pool_2bit if fmt == logan.LOGAN_SEQ_2BIT else batch.pool_u8
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        hp = [pin(x) for x in (pool_np, batch.q_off, batch.q_len, batch.t_off, batch.t_len,
                               batch.q_seed, batch.t_seed)]
        # one compute stream and a ring of three arenas, the library copying each step's
        # inputs ahead on its own stream as soon as the arena is free (options.flags bit 6):
        # every copy overlaps the previous sweeps, and sweeps never overlap each other
        # (C3: 2 streams 25.9 ms per step, 3 streams 25.0, one stream + copy-ahead 23.7;
        # profiles/r02/e2e_probe_v22.txt)
        NE2E = 3
        E2E_COPY_AHEAD = os.environ.get("LOGAN_E2E_COPY_AHEAD", "1") != "0"  # (A/B knob)
        hout = [torch.empty((n_local, 5), dtype=torch.int32).pin_memory().numpy() for _ in range(NE2E)]
        hcells = [torch.empty(n_local, dtype=torch.int64).pin_memory().numpy().view(np.uint64) for _ in range(NE2E)]
        arenas = [logan.HostArena(n_local, batch.pool_len, fmt, db.max_ext_len, device=dev) for _ in range(NE2E)]
        es = torch.cuda.Stream(dev)
        done = [torch.cuda.Event() for _ in range(NE2E)]
        pool_bytes = (batch.pool_len + 3) // 4 if fmt == logan.LOGAN_SEQ_2BIT else batch.pool_len

        stage_ev = None
        if os.environ.get("LOGAN_E2E_DEBUG") == "1":  # per-stage times of the e2e sweeps (debug)
            stage_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * nst)]
            for e in stage_ev:
                e.record(es)

        def e2e_step(s):
            logan.xdrop_batch_host(hp[0], fmt, batch.pool_len, *hp[1:], w.k, w.match, w.mismatch,
                                   w.gap, w.xdrop, arenas[s % NE2E], out=hout[s % NE2E], cells=hcells[s % NE2E],
                                   first_level=first, stream=es, asynchronous=True, subst=subst,
                                   zdrop=args.zdrop, copy_ahead=E2E_COPY_AHEAD, timing_events=stage_ev)
            done[s % NE2E].record(es)

        for s_ in range(NE2E):
            e2e_step(s_)
        torch.cuda.synchronize()
        ke = max(4, args.steps)  # same K as the device-timed steps (steady state)
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()
        e2e_sampler = ClockSampler(sampler.uuid)
        e2e_sampler.start()
        time.sleep(0.1)
        a0 = torch.cuda.Event(enable_timing=True)
        a0.record(es)
        dbg = os.environ.get("LOGAN_E2E_DEBUG") == "1"
        marks, host_t = [], []
        for s_ in range(ke):
            if s_ >= NE2E:
                done[s_ % NE2E].synchronize()  # step s-NE2E's outputs are read before its buffers are reused
                assert int(hcells[s_ % NE2E].sum()) == cells_step
            t0_ = time.perf_counter()
            e2e_step(s_)
            if dbg:
                host_t.append((time.perf_counter() - t0_) * 1e3)
                m = torch.cuda.Event(enable_timing=True)
                m.record(es)
                marks.append(m)
        evx = torch.cuda.Event(enable_timing=True)
        evx.record(es)
        torch.cuda.synchronize()
        e2e_clocks = e2e_sampler.stop()
        e2e_ms = a0.elapsed_time(evx)
        if dbg:
            prev = a0
            per = []
            for m in marks:
                per.append(round(prev.elapsed_time(m), 2))
                prev = m
            print(f"e2e debug: per-step GPU ms {per}; host enqueue ms {[round(x, 2) for x in host_t]}", file=sys.stderr)
            st_ms = {k: round(stage_ev[2 * k].elapsed_time(stage_ev[2 * k + 1]), 2) for k in range(nst)}
            print(f"e2e debug: last step's stage ms {st_ms}; device-timed stage ms "
                  f"{ {k: round(v / args.steps, 2) for k, v in stage_ms.items()} }", file=sys.stderr)
        te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        for k_ in range(NE2E):
            assert int(hcells[k_].sum()) == cells_step
            assert (hout[k_] == out_h).all()  # the host entry point gives the device entry point's results
        e2e = {"value": cells_all * ke / (float(te.item()) / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(pool_bytes + 32 * n_local), "d2h_bytes_per_step": int(28 * n_local),
               "steps": ke, "api": f"logan_xdrop_batch_host_async (one stream, {NE2E} arenas, copy-ahead, pinned)",
               "clocks": e2e_clocks}

    # CPU baseline (rank 0 at N = 1 only) and the parity sample: the oracle on this
    # host's cores over a bounded sample of this rank's pairs, compared element by
    # element with the timed run's output
    cpu = None
    parity = None
    threads = len(os.sched_getaffinity(0))
    if rank == 0:
        rng = np.random.default_rng(2002052000)
        sample_order = rng.permutation(n_local)  # a uniform sample of the pairs, not a prefix
        if world == 1 and share is None and not args.no_cpu_baseline:
            r = oracle_sample(batch, w, args.cpu_seconds, threads, sample_order)
            cpu = {"value": r["cell_sum"] / r["seconds"] / 1e9, "unit": UNIT, "cores": threads,
                   "kind": "oracle", "cpu_model": cpu_model(),
                   "sample": f"{len(r['idx'])} uniformly sampled of the {n_local} pairs ({r['cell_sum']} cells) "
                             f"in {r['seconds']:.1f} s, oracle_pairs on {threads} host threads",
                   "single_thread_c1": single_thread_c1()}
        else:
            r = oracle_sample(batch, w, args.parity_seconds, threads, sample_order)
        sel = r["idx"]
        bad = int(((out_h[sel] != r["out"]).any(axis=1) | (cells_h[sel] != r["cells"])).sum())
        parity = {"pairs": int(len(sel)), "mismatches": bad, "vs": "oracle",
                  "outputs": "score, q_begin, q_end, t_begin, t_end, cells (bit-exact)",
                  "sample": f"uniform sample of {'rank 0' if world > 1 else 'the'} pairs"}

    # N > 1: one gather of the per-pair results to rank 0 (outside the timed region),
    # then rank 0 runs the whole batch alone and compares (partition independence)
    gather_ms = None
    if world > 1:
        cap = max(len(p) for p in parts)
        rec = torch.zeros((cap, 8), dtype=torch.int32, device=dev)
        rec[:n_local, 0:5] = out
        rec[:n_local, 5:7] = cells.view(torch.int32).view(n_local, 2)
        allrec = torch.empty((world * cap, 8), dtype=torch.int32, device=dev)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        dist.all_gather_into_tensor(allrec, rec)
        g1.record(stream)
        torch.cuda.synchronize()
        gather_ms = g0.elapsed_time(g1)
        if rank == 0 and not args.no_verify:
            g = allrec.cpu().numpy().reshape(world, cap, 8)
            full_o = np.zeros((n, 5), np.int32)
            full_c = np.zeros(n, np.uint64)
            for r_, p in enumerate(parts):
                full_o[p] = g[r_, :len(p), 0:5]
                full_c[p] = np.ascontiguousarray(g[r_, :len(p), 5:7]).view(np.uint64).reshape(-1)
            whole = make_batch(args, w, np.arange(n, dtype=np.int64), u8=(args.fmt == "u8"))
            dbw = logan.to_device(whole, fmt, device=dev)
            o1, c1 = logan.xdrop_batch(dbw, w.match, w.mismatch, w.gap, w.xdrop, subst=subst, zdrop=args.zdrop)
            torch.cuda.synchronize()
            o1, c1 = o1.cpu().numpy(), c1.cpu().numpy().view(np.uint64)
            parity["gathered_vs_1gpu"] = {"pairs": n, "mismatches": int(((full_o != o1).any(axis=1) |
                                                                          (full_c != c1)).sum())}
            del dbw

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                # the dominant kernel's arithmetic: int16 pairs (two cells per DPX .S16x2
                # instruction) in the packed windows and the band level, int32 otherwise
                "dtype": "int16x2" if packed else "int32",
                "data": "synthetic (datagen, seeded; DESIGN.md §5)",
                "config": config_dict(w, n, args.fmt + (" (re-encoded to 2-bit on the device each step, logan_pack_2bit)" if u8_packed else ""), args.first_level, world, share),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "parity": parity,
                "gpu_launches": launches_per_step * args.steps, "clocks": clocks,
                "cells_per_step": cells_all, "pairs_this_gpu": n_local,
                "stage_ms_per_step": {str(k): v / args.steps for k, v in stage_ms.items()},
                "levels": {"first": [stats["first_level"], stats["first_width"], stats["first_shape"],
                                     stats["first_helpers"]],
                           "tasks_started": stats["tasks_started"],
                           "tasks_finished": stats["tasks_finished"],
                           "helper_tasks": stats["helper_tasks"],
                           "cells_per_level": stats["cells_per_level"],
                           "window_shifts": stats["window_shifts"]}}
        if gather_ms is not None:
            line["gather_ms"] = gather_ms
        print(json.dumps(line), flush=True)
    ok = parity is None or (parity["mismatches"] == 0 and
                            parity.get("gathered_vs_1gpu", {"mismatches": 0})["mismatches"] == 0)
    if world > 1:
        flag = torch.tensor([0 if ok else 1], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        ok = int(flag.item()) == 0
        dist.destroy_process_group()
    if not ok:
        print("bench.py: the timed output differs from the oracle / the 1-GPU run", file=sys.stderr)
        return 3
    return 0


if __name__ == "__main__":
    sys.exit(main())
