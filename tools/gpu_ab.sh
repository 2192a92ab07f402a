#!/bin/bash
# GPU tests + A/B of library variants: tools/gpu_ab.sh TAG "<test -k expr or ALL>" "<bench args>;<bench args>" name=path ...
TAG=$1; K=$2; BENCHES=$3; shift 3
mkdir -p gpurun_out
if [ "$K" = "ALL" ]; then timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
elif [ "$K" != "NONE" ]; then timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1; fi
tail -3 gpurun_out/${TAG}_pytest.log 2>/dev/null
IFS=';' read -ra BS <<< "$BENCHES"
for b in "${BS[@]}"; do bash tools/ab_bench.sh "$b" "$@"; done > gpurun_out/${TAG}_ab.txt 2>&1
cat gpurun_out/${TAG}_ab.txt
