#!/bin/bash
# Round-end set (one gpurun call): GPU tests, smoke, default bench, other configs, launch list,
# level-1 ncu capture, C6 X-sweep, C7.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
bash tools/gpu_round_profile.sh
for a in "--config 3 --xdrop 20" "--config 4" "--config 5" "--fmt u8" "--zdrop 20"; do
  n=$(echo "$a" | tr -d ' -')
  timeout 600 python bench.py $a --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | grep "^{" > gpurun_out/cfg_$n.json
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 2>/dev/null | grep "^{" > gpurun_out/ref.json
ls -la gpurun_out
