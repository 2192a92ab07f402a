#!/bin/bash
# C6 X-sweep (the paper's read mix, 100K pairs of 2.5-7.5 kb; Tables II-III) with the
# in-tree library: one bench line per X (device-timed, parity-checked) -> gpurun_out/$1.jsonl
OUT=gpurun_out/${1:-c6_xsweep}.jsonl
mkdir -p gpurun_out; : > $OUT
for X in 5 10 20 50 100 200 500 1000 1500 2500 5000; do
  timeout 900 python bench.py --config 6 --xdrop $X --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --parity-seconds 1 2>/dev/null | grep "^{" >> $OUT
done
python -c "
import json
for l in open('$OUT'):
    d=json.loads(l); print('X', d['config']['X'], round(d['value'],1), 'GCUPS', round(d['ms_per_step'],2), 'ms', 'first', d['levels']['first'], 'parity', d['parity']['mismatches'])
"
