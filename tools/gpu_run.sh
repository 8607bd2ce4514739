#!/bin/bash
# Generic gpurun session: run each "name::command" argument, logging to gpurun_out/<tag>/<name>.log
#   gpurun --timeout 1800 -- bash tools/gpu_run.sh <tag> "tests::python -m pytest tests -m gpu -x -q" ...
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > "$OUT/nvidia-smi.csv" 2>&1
for spec in "$@"; do
  name=${spec%%::*}; cmd=${spec#*::}
  start=$(date +%s)
  bash -c "$cmd" > "$OUT/$name.log" 2>&1
  rc=$?
  echo "[$name] rc=$rc $(( $(date +%s) - start ))s" >> "$OUT/summary.txt"
done
echo done > "$OUT/DONE"
