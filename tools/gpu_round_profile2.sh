#!/bin/bash
# Round-2 evidence (one GPU): ncu --set full of the dominant kernel of the default bench
# (C3 X=20) and of C2, the per-launch metrics JSON (profiles/ncu_metrics.json), and the
# launch list of the default bench (gpu__time_duration, cold, serialised).
TAG=${1:-r02}
mkdir -p gpurun_out
for cfg in "3" "2"; do
  python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/b_${cfg}.json 2>/dev/null
  ncu --set full --import-source on --clock-control none -k regex:k_window -c 1 -o gpurun_out/${TAG}_c${cfg} -f \
    python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/${TAG}_c${cfg}_ncu.log 2>&1
  python tools/ncu_metrics.py gpurun_out/${TAG}_c${cfg}.ncu-rep gpurun_out/b_${cfg}.json --out gpurun_out/ncu_metrics.json --tag $TAG
  python tools/ncu_summary.py gpurun_out/${TAG}_c${cfg}.ncu-rep > gpurun_out/${TAG}_ncu_c${cfg}_summary.txt 2>&1
  python tools/ncu_sass_hot.py gpurun_out/${TAG}_c${cfg}.ncu-rep > gpurun_out/${TAG}_ncu_c${cfg}_sass.txt 2>&1
  rm -f gpurun_out/${TAG}_c${cfg}.ncu-rep
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/${TAG}_launches_bench.log 2>&1
ls -la gpurun_out
