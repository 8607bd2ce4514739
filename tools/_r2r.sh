mkdir -p gpurun_out/r2r
for v in 0 1; do SBD_GS_PF=$v timeout 300 python tools/profile_davidson.py 40 > gpurun_out/r2r/dav_gspf$v.json 2>&1; done
timeout 600 python bench.py --no-cpu --no-explicit --no-e2e > gpurun_out/r2r/bench.json 2> gpurun_out/r2r/bench.err
