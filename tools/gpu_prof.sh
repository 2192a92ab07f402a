#!/bin/bash
# ncu captures (one GPU): the dominant k_window launch of a C3 X=20 share 0/8, of the full
# C3 X=20 batch, and of a single long task in the latency shape (tools/latency_probe.py).
TAG=${1:-x}
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_window -c 1 -o gpurun_out/c3_share8_$TAG -f \
  python bench.py --config 3 --share 0/8 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/ncu_c3s8_$TAG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_window -c 1 -o gpurun_out/c3_full_$TAG -f \
  python bench.py --config 3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/ncu_c3_$TAG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_window -s 1 -c 1 -o gpurun_out/lat_$TAG -f \
  python tools/latency_probe.py > gpurun_out/ncu_lat_$TAG.log 2>&1
ls -la gpurun_out/*.ncu-rep
