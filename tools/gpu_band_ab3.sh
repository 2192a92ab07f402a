timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for X in 5000 2500; do
  bash tools/ab_bench.sh "--config 6 --xdrop $X --steps 2 --warmup 3" cap8k=paper_2002_05200_b200/liblogan_xdrop.so cap16k=paper_2002_05200_b200/variants/cap16k.so > gpurun_out/ab3_band_x$X.txt 2>&1
done
