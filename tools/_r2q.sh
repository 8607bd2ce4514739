mkdir -p gpurun_out/r2q
for v in 0 1; do SBD_RES_PF=$v timeout 300 python tools/profile_davidson.py 40 > gpurun_out/r2q/dav_pf$v.json 2>&1; done
