set -x
for X in 10 20 50 100 500 1000 2500 5000; do
  python bench.py --config 6 --xdrop $X --steps 3 --warmup 3 --no-cpu-baseline --stats > gpurun_out/c6_x$X.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_ring -c 1 -o gpurun_out/ring_x5000 python bench.py --config 6 --pairs 10000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_ring.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_window -c 1 -o gpurun_out/l1_c2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l1.log 2>&1
ls -la gpurun_out
