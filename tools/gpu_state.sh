#!/bin/bash
# State check (one gpurun call): GPU tests, smoke, default bench (C3 X=20), C2, and the
# launch list of the default bench. TAG names the outputs.
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
for a in "--config 3 --xdrop 100" "--config 4" "--config 5"; do
  n=$(echo "$a" | tr -d ' -')
  timeout 600 python bench.py $a --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | grep "^{" > gpurun_out/${TAG}_cfg_$n.json
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/${TAG}_launches_bench.log 2>&1
ls -la gpurun_out
