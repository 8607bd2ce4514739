set -u
OUT=gpurun_out/r2o; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:side_kernel_async -s 2 -c 2 -o $OUT/cfg4_side python tools/sigma_probe.py 36 27 30000 2 > $OUT/ncu_cfg4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/cfg4_launches.csv python tools/sigma_probe.py 36 27 30000 2 > /dev/null 2>&1
echo done > $OUT/DONE
