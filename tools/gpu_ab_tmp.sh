timeout 1200 python -m pytest tests -m gpu -x -q -rf > gpurun_out/pytest_pk4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pk4.log; tail -3 gpurun_out/pytest_pk4.log
for a in "--config 3" "--config 2" "--config 3 --share 0/8"; do
  bash tools/ab_bench.sh "$a --steps 10 --warmup 3 --parity-seconds 0.5" cur=paper_2002_05200_b200/liblogan_xdrop.so v7=paper_2002_05200_b200/variants/liblogan_v7.so
done
