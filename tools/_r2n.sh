mkdir -p gpurun_out/r2n
for v in 0 1; do SBD_PAIR_SPLIT=$v timeout 300 python tools/profile_davidson.py 40 > gpurun_out/r2n/dav_split$v.json 2>&1; done
