for X in 5000 1000; do
  bash tools/ab_bench.sh "--config 6 --xdrop $X --first-level 7 --steps 2 --warmup 3" c16=paper_2002_05200_b200/liblogan_xdrop.so v1=paper_2002_05200_b200/variants/v1.so noexact=paper_2002_05200_b200/variants/noexact.so nt64=paper_2002_05200_b200/variants/nt64.so > gpurun_out/ab2_band_x$X.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_band -c 1 -o gpurun_out/band16_x5000 python bench.py --config 6 --pairs 2000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_band16.log 2>&1
