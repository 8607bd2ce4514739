#!/bin/bash
# ncu capture of the Davidson vector kernels at the bench workload (one launch each, k ~ 20).
set -u
TAG=${1:-dav}; OUT=gpurun_out/$TAG; mkdir -p "$OUT"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'residual|gs_|vdots2|rotate' -s 60 -c 5 -o "$OUT/dav" \
    python tools/profile_davidson.py 24 > "$OUT/ncu_dav.log" 2>&1
echo done > "$OUT/DONE"
