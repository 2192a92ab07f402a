#!/bin/bash
# GPU tests + default bench + the small-X lines after the first-window change.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | grep "^{" > gpurun_out/bench_c2.json
for a in "--config 6 --xdrop 5" "--config 6 --xdrop 10" "--config 6 --xdrop 12" "--config 3 --xdrop 10" "--config 3 --xdrop 20"; do
  n=$(echo "$a" | tr -d ' -')
  timeout 300 python bench.py $a --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep "^{" > gpurun_out/cfg_$n.json
done
