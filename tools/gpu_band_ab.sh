# A/B of band-level thread counts on C6, then one ncu capture of k_band (X=5000, 2000 pairs)
for X in 5000 1000; do
  bash tools/ab_bench.sh "--config 6 --xdrop $X --first-level 7 --steps 2 --warmup 3" nt128=paper_2002_05200_b200/liblogan_xdrop.so nt64=paper_2002_05200_b200/variants/nt64.so nt256=paper_2002_05200_b200/variants/nt256.so > gpurun_out/ab_band_x$X.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_band -c 1 -o gpurun_out/band_x5000 python bench.py --config 6 --pairs 2000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_band.log 2>&1
