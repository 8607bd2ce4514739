#!/bin/bash
# One gpurun session: GPU tests, smoke, bench, ncu launch list + full capture of the sigma kernels.
#   gpurun --timeout 2400 -- bash tools/gpu_session.sh [tag]
# Outputs land in gpurun_out/<tag>/ (merged back by gpurun).
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
cp -f MEASURED_PEAKS.json "$OUT/" 2>/dev/null
python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
# launch list (cold-cache, serialised): one sigma pass, shares only
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-davidson --no-cpu --no-e2e \
    > "$OUT/launches_bench.log" 2>&1
# full capture of the sigma kernels (one launch each, after warm-up)
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'side_kernel|cross_kernel|transpose_kernel' -s 12 -c 4 -o "$OUT/sigma" \
    python bench.py --steps 1 --warmup 3 --no-davidson --no-cpu --no-e2e > "$OUT/ncu_full.log" 2>&1
# Davidson: per-phase device/host time, then one ncu capture of each vector pass
timeout 600 python tools/profile_davidson.py > "$OUT/dav_profile.json" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'residual|gs_|vdots2|rotate' -s 60 -c 5 -o "$OUT/dav" \
    python tools/profile_davidson.py 24 > "$OUT/ncu_dav.log" 2>&1
# keep the merged-back output under gpurun's 64 MiB: summarise the Davidson capture on the box
python tools/ncu_summary.py "$OUT/dav.ncu-rep" > "$OUT/ncu_davidson_full.jsonl" 2>/dev/null && rm -f "$OUT/dav.ncu-rep"
python tools/ncu_summary.py "$OUT/sigma.ncu-rep" > "$OUT/ncu_sigma_full.jsonl" 2>/dev/null
echo done > "$OUT/DONE"
