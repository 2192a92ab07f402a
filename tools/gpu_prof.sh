#!/bin/bash
# ncu captures (one GPU): the dominant k_window launch of a C3 X=20 share 0/8, of the full
# C3 X=20 batch, and of a single long task in the latency shape (tools/latency_probe.py).
# Summaries are written next to the reports; only the reports named in KEEP stay (64 MiB cap).
TAG=${1:-x}
KEEP=${2:-none}
mkdir -p gpurun_out
summ() {
  python tools/ncu_summary.py gpurun_out/$1.ncu-rep > gpurun_out/$1_summary.txt 2>&1
  python tools/ncu_stalls.py gpurun_out/$1.ncu-rep 30 > gpurun_out/$1_stalls.txt 2>&1
  python tools/ncu_sass_hot.py gpurun_out/$1.ncu-rep > gpurun_out/$1_sass.txt 2>&1
  python tools/ncu_stall_agg.py gpurun_out/$1.ncu-rep ${2:-1000} >> gpurun_out/$1_stalls.txt 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/$1_source.csv 2>/dev/null
  gzip -f gpurun_out/$1_source.csv
  case " $KEEP " in *" $1 "*) ;; *) rm -f gpurun_out/$1.ncu-rep ;; esac
}
ncu --set full --import-source on --clock-control none -k regex:k_window -c 1 -o gpurun_out/c3_share8_$TAG -f \
  python bench.py --config 3 --share 0/8 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/ncu_c3s8_$TAG.log 2>&1
summ c3_share8_$TAG 500000
ncu --set full --import-source on --clock-control none -k regex:k_window -c 1 -o gpurun_out/c3_full_$TAG -f \
  python bench.py --config 3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/ncu_c3_$TAG.log 2>&1
summ c3_full_$TAG 1000000
ncu --set full --import-source on --clock-control none -k regex:k_window -s 1 -c 1 -o gpurun_out/lat_$TAG -f \
  python tools/latency_probe.py > gpurun_out/ncu_lat_$TAG.log 2>&1
summ lat_$TAG 10000
ls -la gpurun_out/
