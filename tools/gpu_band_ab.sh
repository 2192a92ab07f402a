#!/bin/bash
# Band-level variants: band parity tests per variant, then C6 A/B at X = 2500 / 5000.
mkdir -p gpurun_out
for nv in "$@"; do
  name=${nv%%=*}; lib=${nv#*=}
  LOGAN_LIB=$lib timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "band or wide or large_x or xsweep or x_sweep" 2>&1 | tail -1 | sed "s/^/$name pytest: /"
done
bash tools/ab_bench.sh "--config 6 --xdrop 5000 --pairs 20000 --steps 3 --warmup 2" "$@"
bash tools/ab_bench.sh "--config 6 --xdrop 2500 --pairs 20000 --steps 3 --warmup 2" "$@"
bash tools/ab_bench.sh "--config 6 --xdrop 1500 --pairs 20000 --steps 3 --warmup 2" "$@"
bash tools/ab_bench.sh "--config 6 --xdrop 10000 --pairs 10000 --steps 2 --warmup 1" "$@"
