# correctness of the wide-band level first (bounded), then the whole GPU suite, then C6 timings
set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "ring or exhaustive" > gpurun_out/band_tests.log 2>&1; echo "rc=$?" >> gpurun_out/band_tests.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for X in 5000 2500 1000 500; do
  timeout 300 python bench.py --config 6 --xdrop $X --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --stats > gpurun_out/c6b_x$X.log 2>&1
done
for X in 1000 500; do
  timeout 300 python bench.py --config 6 --xdrop $X --first-level 7 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --stats > gpurun_out/c6b_x${X}_l7.log 2>&1
done
