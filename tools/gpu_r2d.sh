set -u
OUT=gpurun_out/r2d; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "direct_ci or sigma_variants" > $OUT/dci_tests.log 2>&1
for v in 0 1; do SBD_CROSS_DCI=$v timeout 120 python tools/sigma_probe.py 12 6 0 20 >> $OUT/cfg1_ab.log 2>&1; done
for v in 0 1; do SBD_CROSS_DCI=$v timeout 120 python tools/sigma_probe.py 12 6 0 20 >> $OUT/cfg1_ab.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $OUT/cfg1_launches.csv python tools/sigma_probe.py 12 6 0 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cross_kernel_dci -s 2 -c 1 -o $OUT/dci python tools/sigma_probe.py 12 6 0 2 > $OUT/ncu_dci.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scale_parity.py -x -q -rA -k "ground_state" > $OUT/scale.log 2>&1
for v in 0 1 2 3 4 5 6 7; do SAN_VARIANT=$v timeout 300 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 3 python tools/sanitize_cases.py sigma > $OUT/racecheck_sigma_$v.log 2>&1; done
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 5 python tools/sanitize_cases.py davidson > $OUT/racecheck_davidson.log 2>&1
for c in explicit ingest dense; do timeout 300 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 5 python tools/sanitize_cases.py $c > $OUT/racecheck_$c.log 2>&1; done
echo done > $OUT/DONE
