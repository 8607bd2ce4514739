mkdir -p gpurun_out/r2m
for v in 0 1 2 3; do SBD_PAIR_SPLIT=$v timeout 300 python tools/profile_davidson.py 40 > gpurun_out/r2m/dav_split$v.json 2>&1; done
timeout 1200 python -m pytest tests/test_gpu_davidson.py tests/test_gpu_distributed.py tests/test_gpu_explicit.py -m gpu -x -q --timeout 300 > gpurun_out/r2m/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2m/pytest_gpu.log
