#!/bin/bash
# Round evidence on one GPU: GPU tests, smoke, default bench (C3 X=20) and C2 with the CPU
# baseline, ncu --set full of the dominant kernel of both (+ the integer-instruction
# metric), the per-launch metrics JSON, SASS histogram, and the launch list of the default bench.
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err
timeout 600 python bench.py --config 2 > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
for cfg in "3" "2"; do
  python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/b_${cfg}.json 2>/dev/null
  ncu --set full --import-source on --clock-control none -k regex:k_window -c 1 -o gpurun_out/${TAG}_c${cfg} -f \
    python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/${TAG}_c${cfg}_ncu.log 2>&1
  ncu --metrics smsp__sass_thread_inst_executed_op_integer_pred_on.sum,smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:k_window -c 1 -o gpurun_out/${TAG}_c${cfg}_int -f \
    python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/${TAG}_c${cfg}_int.log 2>&1
  python tools/ncu_metrics.py gpurun_out/${TAG}_c${cfg}.ncu-rep gpurun_out/b_${cfg}.json --int-rep gpurun_out/${TAG}_c${cfg}_int.ncu-rep --out gpurun_out/ncu_metrics.json --tag $TAG
  python tools/ncu_summary.py gpurun_out/${TAG}_c${cfg}.ncu-rep > gpurun_out/${TAG}_ncu_c${cfg}_summary.txt 2>&1
  python tools/ncu_sass_hot.py gpurun_out/${TAG}_c${cfg}.ncu-rep > gpurun_out/${TAG}_ncu_c${cfg}_sass.txt 2>&1
  rm -f gpurun_out/${TAG}_c${cfg}.ncu-rep gpurun_out/${TAG}_c${cfg}_int.ncu-rep
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --parity-seconds 0.3 > gpurun_out/${TAG}_launches_bench.log 2>&1
ls -la gpurun_out
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
for a in "--config 3 --xdrop 10" "--config 3 --xdrop 50" "--config 3 --xdrop 100" "--config 4" "--config 5" "--fmt u8" "--zdrop 20" "--config 6 --xdrop 5000"; do
  n=$(echo "$a" | tr -d ' -')
  timeout 900 python bench.py $a --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | grep "^{" > gpurun_out/${TAG}_cfg_$n.json
done
