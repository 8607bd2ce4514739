set -u
OUT=gpurun_out/r2t; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "direct_ci" > $OUT/tests.log 2>&1
timeout 300 python tools/ab_env.py SBD_CROSS_DCI=0 SBD_DCI_WS=0 SBD_DCI_WS=1 --points cfg1 --steps 20 > $OUT/ab_dci.jsonl 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cross_kernel_dci -s 2 -c 1 -o $OUT/dci python tools/sigma_probe.py 12 6 0 2 > $OUT/ncu_dci.log 2>&1
echo done > $OUT/DONE
