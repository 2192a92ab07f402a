#!/bin/bash
# A/B of library variants on strong-scaling shares (one box, alternating runs).
mkdir -p gpurun_out
for a in "--config 3 --share 0/8" "--config 2 --share 0/8" "--config 5 --share 0/8" "--config 3"; do
  bash tools/ab_bench.sh "$a --steps 5 --warmup 2 --parity-seconds 0.5" main=paper_2002_05200_b200/liblogan_xdrop.so "$@"
done
timeout 600 python tools/latency_probe.py > gpurun_out/latency_probe_ab.txt 2>&1
