#!/bin/bash
# Line-level ncu capture of the first-level kernel of one bench config: per-source-line
# executed instructions (tools/ncu_lines.py), the opcode histogram and the summary.
TAG=${1:-r02}; CFG=${2:-3}; shift 2; EXTRA="$@"
mkdir -p gpurun_out
python bench.py --config $CFG $EXTRA --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/${TAG}_b.json 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:k_window -c 1 -o gpurun_out/${TAG} -f \
  python bench.py --config $CFG $EXTRA --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/${TAG}_ncu.log 2>&1
python tools/ncu_lines.py gpurun_out/${TAG}.ncu-rep 120 > gpurun_out/${TAG}_lines.txt 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}.ncu-rep > gpurun_out/${TAG}_summary.txt 2>&1
python tools/ncu_sass_hot.py gpurun_out/${TAG}.ncu-rep > gpurun_out/${TAG}_sass.txt 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sasssrc.csv 2>/dev/null
gzip -f gpurun_out/${TAG}_sasssrc.csv
rm -f gpurun_out/${TAG}.ncu-rep
ls -la gpurun_out
