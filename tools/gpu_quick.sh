#!/bin/bash
# Quick gpurun: GPU tests + bench + one ncu capture of a kernel regex.
#   gpurun -- bash tools/gpu_quick.sh <tag> [kernel-regex] [pytest-args]
set -u
TAG=${1:-q}; KRE=${2:-}; PYARGS=${3:-tests}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
timeout 1200 python -m pytest $PYARGS -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"
if [ -n "$KRE" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 3 -c 2 -o "$OUT/prof" \
    python bench.py --steps 1 --warmup 3 --no-davidson --no-cpu --no-e2e > "$OUT/ncu.log" 2>&1
fi
echo done > "$OUT/DONE"
