#!/bin/bash
# Line-level ncu capture of the band level (k_band) at a given X on C6 (the paper's read mix).
TAG=${1:-band}; X=${2:-5000}; PAIRS=${3:-10000}
mkdir -p gpurun_out
python bench.py --config 6 --xdrop $X --pairs $PAIRS --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --parity-seconds 0.5 > gpurun_out/${TAG}_b.json 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:k_band -c 1 -o gpurun_out/${TAG} -f \
  python bench.py --config 6 --xdrop $X --pairs $PAIRS --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/${TAG}_ncu.log 2>&1
python tools/ncu_lines.py gpurun_out/${TAG}.ncu-rep 150 > gpurun_out/${TAG}_lines.txt 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}.ncu-rep > gpurun_out/${TAG}_summary.txt 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sasssrc.csv 2>/dev/null
gzip -f gpurun_out/${TAG}_sasssrc.csv
rm -f gpurun_out/${TAG}.ncu-rep
