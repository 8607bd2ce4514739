set -u
OUT=gpurun_out/r2v; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q -k "sigma_variants or direct_ci or big_config or random_instances" > $OUT/tests.log 2>&1
timeout 300 python tools/ab_env.py SBD_DENSE_GEMM=0 SBD_DENSE_GEMM=1 --points cfg1,1e6 --steps 20 > $OUT/ab_dense.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $OUT/cfg1_launches.csv python tools/sigma_probe.py 12 6 0 2 > /dev/null 2>&1
timeout 300 python tools/cfg1_davidson.py > $OUT/cfg1_davidson.json 2>&1
echo done > $OUT/DONE
