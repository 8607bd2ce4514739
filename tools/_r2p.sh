mkdir -p gpurun_out/r2p
for v in 1 2 4; do SBD_RES_SPLIT=$v timeout 300 python tools/profile_davidson.py 40 > gpurun_out/r2p/dav_res$v.json 2>&1; done
SBD_RES_SPLIT=4 timeout 300 python tools/profile_davidson.py 40 3 > gpurun_out/r2p/dav3_res4.json 2>&1
timeout 1200 python -m pytest tests/test_gpu_davidson.py tests/test_gpu_distributed.py -m gpu -x -q --timeout 300 > gpurun_out/r2p/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2p/pytest_gpu.log
