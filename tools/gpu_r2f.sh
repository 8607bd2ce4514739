set -u
OUT=gpurun_out/r2f; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_davidson.py -x -q -k "direct_ci or sigma_variants or native_driver or selective or large_subspace" > $OUT/tests.log 2>&1
timeout 300 python tools/ab_env.py SBD_CROSS_DCI=0 SBD_CROSS_DCI=1 --points cfg1 --steps 20 > $OUT/ab_dci.jsonl 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cross_kernel_dci -s 2 -c 1 -o $OUT/dci python tools/sigma_probe.py 12 6 0 2 > $OUT/ncu_dci.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/cfg1_launches.csv python tools/sigma_probe.py 12 6 0 2 > /dev/null 2>&1
timeout 900 python bench.py --no-cpu --steps 20 > $OUT/bench.json 2> $OUT/bench.err
timeout 1500 python tools/cfg4_solve.py --check > $OUT/cfg4_solve.jsonl 2> $OUT/cfg4_solve.err
echo done > $OUT/DONE
