#!/usr/bin/env python
"""Per-launch ncu counters of the dominant kernel of a bench run, for the
roofline object of bench.py (profiles/ncu_metrics.json).

    python tools/ncu_metrics.py REPORT.ncu-rep BENCH.json [--out profiles/ncu_metrics.json]

REPORT is an `ncu --set full -k regex:k_window -c 1` capture of
`bench.py --steps 1 --warmup 0 ...` (the first k_window launch is bench's
untimed stats run: the same work as every timed step); BENCH.json is that
run's JSON line (it names the workload and the cells of the captured level).
"""
import argparse
import csv
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "duration_ns": "gpu__time_duration.sum",
    "warp_inst": "smsp__inst_executed.sum",
    "int_thread_inst": "smsp__sass_thread_inst_executed_op_integer_pred_on.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm_clock_hz": "sm__cycles_elapsed.avg.per_second",
    "registers": "launch__registers_per_thread",
}
UNIT_SCALE = {"ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
              "hz": 1.0, "khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "MHz": 1e6, "GHz": 1e9}


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(hdr)}
    res = {"kernel": vals[col["Kernel Name"]] if "Kernel Name" in col else ""}
    for k, m in METRICS.items():
        if m not in col:
            continue
        v = float(vals[col[m]].replace(",", ""))
        res[k] = v * UNIT_SCALE.get(units[col[m]], 1.0)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("bench_json")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_metrics.json"))
    ap.add_argument("--tag", default="")
    ap.add_argument("--int-rep", default=None,
                    help="a second capture of the same launch with --metrics "
                         "smsp__sass_thread_inst_executed_op_integer_pred_on.sum (not in --set full)")
    args = ap.parse_args()
    line = json.loads([ln for ln in open(args.bench_json) if ln.startswith("{")][-1])
    cfg = line["config"]
    level = line["levels"]["first"][0]
    cells = line["levels"]["cells_per_level"][level - 1]
    m = raw_metrics(args.rep)
    if args.int_rep and os.path.exists(args.int_rep):
        mi = raw_metrics(args.int_rep)
        if "int_thread_inst" in mi:
            m["int_thread_inst"] = mi["int_thread_inst"]
    dur = m["duration_ns"] * 1e-9
    entry = {
        "kernel": m["kernel"], "level": level, "cells_per_launch": cells,
        "duration_ms_ncu": m["duration_ns"] * 1e-6,
        "dram_bytes": int(m.get("dram_read", 0) + m.get("dram_write", 0)),
        "sass_thread_inst_per_cell": m["warp_inst"] * 32 / cells,
        "int_thread_inst_per_cell": m.get("int_thread_inst", 0) / cells,
        "int_warp_gips": m.get("int_thread_inst", 0) / 32 / dur / 1e9,
        "warp_gips": m["warp_inst"] / dur / 1e9,
        "alu_pipe_pct": m.get("alu_pipe_pct"), "fma_pipe_pct": m.get("fma_pipe_pct"),
        "issue_pct": m.get("issue_pct"), "registers": m.get("registers"),
        "source": f"{os.path.basename(args.rep)} (ncu --set full, --clock-control none) {args.tag} "
                  f"{time.strftime('%Y-%m-%d')}",
    }
    key = f"{cfg['workload']}/{cfg['fmt']}/level{level}"
    db = json.load(open(args.out)) if os.path.exists(args.out) else {}
    db[key] = entry
    json.dump(db, open(args.out, "w"), indent=1, sort_keys=True)
    print(key, json.dumps(entry))


if __name__ == "__main__":
    sys.exit(main())
