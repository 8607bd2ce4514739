set -u
OUT=gpurun_out/r2q; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "sigma_variants" > $OUT/tests.log 2>&1
timeout 900 python tools/ab_env.py SBD_CONN_WINDOW=0 SBD_CONN_WINDOW=1 --points cfg1,1e6,1e7,cfg2,3e8,cfg4,1e9 > $OUT/ab_cwin.jsonl 2> $OUT/ab_cwin.err
echo done > $OUT/DONE
