#!/usr/bin/env python
"""Build and run the integer-throughput microbenchmark (tools/int_peak.cu) and
write profiles/int_peak.json, the measured peak bench.py's roofline divides by.

    python tools/int_peak.py [--out profiles/int_peak.json]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "int_peak.json"))
    args = ap.parse_args()
    exe = "/tmp/logan_int_peak"
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "-o", exe, os.path.join(HERE, "int_peak.cu")])
    runs = [json.loads(subprocess.check_output([exe], text=True)) for _ in range(3)]
    r = runs[-1]
    rate = {k: statistics.median(x["inst_per_clk_per_sm"][k] for x in runs) for k in r["inst_per_clk_per_sm"]}
    alu = [rate[k] for k in ("VIMNMX3", "VIADDMNMX", "VIMNMX.U32", "LOP3", "SHF")]
    out = {
        "gpu": r["gpu"], "sms": r["sms"], "threads_per_sm": r["threads_per_sm"],
        "inst_per_clk_per_sm": rate,
        "alu_int32_ops_per_clk_per_sm": round(min(alu), 2),
        "fma_int32_ops_per_clk_per_sm": round(rate["IMAD"], 2),
        "issue_inst_per_clk_per_sm": round(rate["VIMNMX3+IMAD (1:1)"], 2),
        "s16x2_ops_per_clk_per_sm": round(2 * min(rate["VIMNMX3.S16x2"], rate["VIADDMNMX.S16x2"]), 2),
        "source": "tools/int_peak.cu (clock64 per block, 32 warps/SM, 8 independent chains/thread), "
                  f"median of 3 runs, {time.strftime('%Y-%m-%d')}",
        "note": "alu = min over the cell's ALU-pipe forms (VIMNMX3, VIADDMNMX, VIMNMX.U32, LOP3, SHF); "
                "issue = VIMNMX3 and IMAD interleaved 1:1 (ALU and FMA pipes together); s16x2 counts 2 lanes/op",
    }
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
