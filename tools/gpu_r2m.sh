set -u
OUT=gpurun_out/r2m; mkdir -p $OUT
timeout 900 python tools/ab_env.py SBD_SIDE_RING=3 SBD_SIDE_RING=4 SBD_SIDE_RING=6 --points cfg1,1e6,1e7,cfg2,3e8,cfg4,1e9 > $OUT/ab_ring.jsonl 2> $OUT/ab_ring.err
echo done > $OUT/DONE
