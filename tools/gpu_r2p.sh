set -u
OUT=gpurun_out/r2p; mkdir -p $OUT
timeout 900 python tools/ab_env.py SBD_L2_HINTS=0 SBD_L2_HINTS=1 --points cfg1,1e6,1e7,cfg2,3e8,cfg4,1e9 > $OUT/ab_hints.jsonl 2> $OUT/ab_hints.err
SBD_L2_HINTS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file $OUT/cfg4_launches_hints.csv python tools/sigma_probe.py 36 27 30000 2 > /dev/null 2>&1
echo done > $OUT/DONE
