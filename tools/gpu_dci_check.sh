# direct-CI kernel check: its tests, cfg1 sigma with/without it, and its launch time
set -u
OUT=gpurun_out/${1:-dci}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "direct_ci" > $OUT/tests.log 2>&1
timeout 300 python tools/ab_env.py SBD_CROSS_DCI=0 SBD_CROSS_DCI=1 --points cfg1 --steps 30 > $OUT/ab_dci.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $OUT/cfg1_launches.csv python tools/sigma_probe.py 12 6 0 2 > /dev/null 2>&1
echo done > $OUT/DONE
