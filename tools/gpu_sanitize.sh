#!/bin/bash
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
{ echo "== san_mem"; timeout 900 $S --tool memcheck python tools/sanitize_run.py 2>&1 | tail -4
  echo "== san_race"; timeout 900 $S --tool racecheck python tools/sanitize_run.py --small 2>&1 | tail -4
  echo "== san_sync"; timeout 900 $S --tool synccheck python tools/sanitize_run.py --small 2>&1 | tail -4; } > gpurun_out/sanitizer.txt
