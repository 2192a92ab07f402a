#!/bin/bash
# ncu --set full of the dominant k_window launch of a bench configuration, summarised on the box.
# usage: bash tools/gpu_prof2.sh TAG "<bench args>" [KEEP=1]
TAG=$1; ARGS=$2; KEEP=${3:-0}
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_window -c 1 -o gpurun_out/$TAG -f \
  python bench.py $ARGS --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/$TAG.ncu-rep > gpurun_out/${TAG}_summary.txt 2>&1
python tools/ncu_sass_hot.py gpurun_out/$TAG.ncu-rep > gpurun_out/${TAG}_sass.txt 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${TAG}_source.csv.gz
[ "$KEEP" = "1" ] || rm -f gpurun_out/$TAG.ncu-rep
