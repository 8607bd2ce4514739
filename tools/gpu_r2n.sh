set -u
OUT=gpurun_out/r2n; mkdir -p $OUT
timeout 900 python tools/sweep.py --steps 10 > $OUT/sweep.json 2> $OUT/sweep.err
timeout 600 python tools/cfg1_davidson.py > $OUT/cfg1_davidson.json 2> $OUT/cfg1_davidson.err
echo done > $OUT/DONE
