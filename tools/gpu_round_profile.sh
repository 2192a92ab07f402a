#!/bin/bash
# Round-end measurement set (one gpurun call): default bench, launch list, level-1 ncu capture,
# the C6 X-sweep and the protein-like C7 line.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_window -c 1 -o gpurun_out/l1_c2 \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l1.log 2>&1
for X in 10 20 50 100 500 1000 2500 5000; do
  python bench.py --config 6 --xdrop $X --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep "^{" > gpurun_out/c6_x$X.json
done
python bench.py --config 7 --steps 10 --warmup 3 2>/dev/null | grep "^{" > gpurun_out/c7.json
ls -la gpurun_out
