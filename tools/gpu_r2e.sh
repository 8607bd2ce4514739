set -u
OUT=gpurun_out/r2e; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "sigma_variants or direct_ci" > $OUT/kernel_tests.log 2>&1
timeout 300 python tools/ab_env.py SBD_CROSS_DCI=0 SBD_CROSS_DCI=1 --points cfg1 --steps 20 > $OUT/ab_dci.jsonl 2>&1
V='SBD_SIDE_PERSIST=0 SBD_SIDE_PERSIST=1 SBD_SIDE_PERSIST=0,SBD_PERM_BETA=1 SBD_SIDE_PERSIST=0,SBD_PERM_BETA=1,SBD_SIDE_CA=1 SBD_SIDE_PERSIST=0,SBD_SIDE_CA=1 SBD_SIDE_PERSIST=1,SBD_SIDE_CA=1'
timeout 900 python tools/ab_env.py $V --points cfg1,1e6,1e7,cfg2,3e8,cfg4,1e9 > $OUT/ab_sorted.jsonl 2> $OUT/ab_sorted.err
SBD_CONN_SORT=0 timeout 600 python tools/ab_env.py SBD_SIDE_PERSIST=0 SBD_SIDE_PERSIST=1 --points cfg1,cfg2,cfg4,1e9 > $OUT/ab_unsorted.jsonl 2> $OUT/ab_unsorted.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cross_kernel_dci -s 2 -c 1 -o $OUT/dci python tools/sigma_probe.py 12 6 0 2 > $OUT/ncu_dci.log 2>&1
for v in 0 3; do SAN_VARIANT=$v timeout 300 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 3 python tools/sanitize_cases.py sigma > $OUT/racecheck_sigma_$v.log 2>&1; done
echo done > $OUT/DONE
