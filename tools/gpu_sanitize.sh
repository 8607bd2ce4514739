# compute-sanitizer over every kernel variant (tools/sanitize_cases.py), one racecheck process per sigma variant
set -u
OUT=gpurun_out/${1:-sanitize}; mkdir -p $OUT
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_cases.py > $OUT/memcheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_cases.py > $OUT/synccheck.log 2>&1
for v in 1 2 4 6 7 8 9; do SAN_VARIANT=$v timeout 400 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 5 python tools/sanitize_cases.py sigma > $OUT/racecheck_sigma_$v.log 2>&1; done
for c in explicit ingest dense residual tables128; do timeout 300 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 5 python tools/sanitize_cases.py $c > $OUT/racecheck_$c.log 2>&1; done
echo done > $OUT/DONE
