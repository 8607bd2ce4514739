mkdir -p gpurun_out/r2s
timeout 300 python tools/profile_davidson.py 40 > gpurun_out/r2s/dav.json 2>&1
timeout 600 python bench.py --no-cpu --no-explicit --no-e2e > gpurun_out/r2s/bench.json 2> gpurun_out/r2s/bench.err
timeout 1200 python -m pytest tests/test_gpu_davidson.py tests/test_gpu_distributed.py -m gpu -x -q --timeout 300 > gpurun_out/r2s/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2s/pytest_gpu.log
