set -u
OUT=gpurun_out/r2h; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "direct_ci or sigma_variants or davidson_passes" > $OUT/tests.log 2>&1
timeout 300 python tools/ab_env.py SBD_CROSS_DCI=0 SBD_CROSS_DCI=1 --points cfg1 --steps 20 > $OUT/ab_dci.jsonl 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cross_kernel_dci -s 2 -c 1 -o $OUT/dci python tools/sigma_probe.py 12 6 0 2 > $OUT/ncu_dci.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/cfg1_launches.csv python tools/sigma_probe.py 12 6 0 2 > /dev/null 2>&1
timeout 900 python tools/ab_davidson.py SBD_RES_KEEPV=0 SBD_RES_KEEPV=1 > $OUT/ab_keepv.json 2>&1
echo done > $OUT/DONE
