# one-off A/B session: tests (pytest -k expression) then tools/ab_env.py variants over sweep points
#   bash tools/gpu_ab.sh <tag> "<pytest -k expr>" "<points>" VAR=.. VAR=..
set -u
TAG=$1; K=$2; PTS=$3; shift 3
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q -k "$K" > $OUT/tests.log 2>&1
timeout 1200 python tools/ab_env.py "$@" --points "$PTS" > $OUT/ab.jsonl 2> $OUT/ab.err
echo done > $OUT/DONE
