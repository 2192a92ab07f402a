#!/usr/bin/env python
"""Projected strong scaling on ONE GPU: every share of an N-way split.

For each workload, runs ``bench.py`` on the whole batch (N = 1) and on every
share r of the N-way LPT split (``--share r/N``) for N in {2, 4, 8}, one after
the other on the same GPU, and reports per-share device times.  An N-GPU run's
step time is the max over ranks, so the projected N-GPU throughput is
total cells / max_r T_r and the projected efficiency T_1 / (N * max_r T_r).

    python tools/strong_scaling.py [--out profiles/r02_strong_scaling.json] [--only c3_x20,...]
"""
from __future__ import annotations

import argparse
import contextlib
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

WORKLOADS = {
    "c3_x20": ["--config", "3", "--xdrop", "20"],
    "c3_x50": ["--config", "3", "--xdrop", "50"],
    "c3_x100": ["--config", "3", "--xdrop", "100"],
    "c2_x20": ["--config", "2"],
    "c5_x100": ["--config", "5"],
}
COMMON = ["--no-e2e", "--no-cpu-baseline", "--parity-seconds", "1", "--steps", "5", "--warmup", "3"]


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = bench.main(argv)
    lines = [ln for ln in buf.getvalue().splitlines() if ln.startswith("{")]
    if rc != 0 or not lines:
        raise RuntimeError(f"bench {argv} failed (rc={rc})")
    return json.loads(lines[-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "strong_scaling.json"))
    ap.add_argument("--only", default=None)
    ap.add_argument("--ns", default="2,4,8")
    args = ap.parse_args()
    names = args.only.split(",") if args.only else list(WORKLOADS)
    ns = [int(x) for x in args.ns.split(",")]
    res = {}
    for name in names:
        base = WORKLOADS[name] + COMMON
        full = run(base)
        t1 = full["ms_per_step"]
        entry = {"cells": full["cells_per_step"], "ms_1gpu": t1, "gcups_1gpu": full["value"],
                 "first": full["levels"]["first"], "shares": {}}
        for n in ns:
            shares = [run(base + ["--share", f"{r}/{n}"]) for r in range(n)]
            ms = [s["ms_per_step"] for s in shares]
            cells = sum(s["cells_per_step"] for s in shares)
            assert cells == full["cells_per_step"], (name, n, cells, full["cells_per_step"])
            tmax = max(ms)
            entry["shares"][str(n)] = {
                "ms_per_share": ms, "ms_max": tmax, "pairs": [s["pairs_this_gpu"] for s in shares],
                "first": [s["levels"]["first"] for s in shares],
                "projected_gcups": cells / (tmax / 1e3) / 1e9,
                "projected_efficiency": t1 / (n * tmax),
                "parity_mismatches": sum(s["parity"]["mismatches"] for s in shares)}
            print(f"{name} N={n}: share ms {['%.2f' % x for x in ms]} -> eff {t1 / (n * tmax):.3f}",
                  file=sys.stderr, flush=True)
        res[name] = entry
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        json.dump(res, open(args.out, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
