#!/bin/bash
# A/B of library variants on one box: tools/ab_bench.sh "<bench args>" name=path ...
args="$1"; shift
mkdir -p gpurun_out
echo "== $args"
for rep in 1 2; do
  for nv in "$@"; do
    name=${nv%%=*}; lib=${nv#*=}
    LOGAN_LIB=$lib python bench.py $args --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('$name rep$rep', round(d['value'],1), 'GCUPS', round(d['ms_per_step'],3), 'ms', 'kernel', round(r['kernel_ms'],3))
"
  done
done
