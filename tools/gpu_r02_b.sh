#!/bin/bash
# Latency diagnostics: instruction latencies, integer peaks, per-antidiagonal latency of each
# shape, and an ncu capture of the dominant kernel of a strong-scaling share (C2, share 0/8).
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat_probe tools/lat_probe.cu && /tmp/lat_probe > gpurun_out/lat_probe.json 2>&1
timeout 300 python tools/int_peak.py --out gpurun_out/int_peak.json > gpurun_out/int_peak.log 2>&1
timeout 600 python tools/latency_probe.py > gpurun_out/latency_probe.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_window -c 1 -o gpurun_out/c2_share8 -f \
  python bench.py --config 2 --share 0/8 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --parity-seconds 0.5 > gpurun_out/ncu_c2_share8.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_window -c 1 -o gpurun_out/c3_full -f \
  python bench.py --config 3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --parity-seconds 0.5 > gpurun_out/ncu_c3_full.log 2>&1
ls -la gpurun_out
