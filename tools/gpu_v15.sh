#!/bin/bash
# GPU tests + default bench + the X-sweep and C3 lines after the first-window threshold change.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py 2>/dev/null | grep "^{" > gpurun_out/bench_c2.json
for X in 5 10 12 18 20 50 100 500 1000 2500 5000; do
  timeout 300 python bench.py --config 6 --xdrop $X --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep "^{" > gpurun_out/c6_x$X.json
done
for X in 10 20; do
  timeout 300 python bench.py --config 3 --xdrop $X --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep "^{" > gpurun_out/c3_x$X.json
done
