#!/bin/bash
# Generic check call: GPU tests (stop on first failure), then the default bench, the C2
# bench, the latency probe and the 8-way strong-scaling shares of C2 / C3 X=20.
# usage: bash tools/gpu_check.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -rf > gpurun_out/pytest_$TAG.log 2>&1; rc=$?
echo "pytest rc=$rc" >> gpurun_out/pytest_$TAG.log
tail -5 gpurun_out/pytest_$TAG.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench_c2_$TAG.json 2> gpurun_out/bench_c2_$TAG.err
timeout 600 python tools/latency_probe.py > gpurun_out/latency_probe_$TAG.txt 2>&1
timeout 1200 python tools/strong_scaling.py --only c2_x20,c3_x20,c5_x100 --ns 8 --out gpurun_out/strong_$TAG.json > /dev/null 2> gpurun_out/strong_$TAG.err
tail -3 gpurun_out/strong_$TAG.err
python - <<PY
import json
for f in ("gpurun_out/bench_c3_$TAG.json", "gpurun_out/bench_c2_$TAG.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"], 1), round(d["ms_per_step"], 3), round(d["roofline"]["frac"], 3), d["parity"])
    except Exception as e:
        print(f, "failed", e)
PY
