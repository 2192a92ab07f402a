#!/bin/bash
# A/B of two libraries over the C6 X-sweep (window levels) and C2: tools/ab_sweep.sh new.so base.so
for X in 10 20 50 100 500 1000; do
  bash tools/ab_bench.sh "--config 6 --xdrop $X --pairs 50000 --steps 4 --warmup 2" new=$1 base=$2 | sed "s/^/X=$X /"
done
bash tools/ab_bench.sh "--steps 10 --warmup 3" new=$1 base=$2 | sed "s/^/C2 /"
