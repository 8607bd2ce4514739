set -u
OUT=gpurun_out/r2i; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "direct_ci or sigma_variants or davidson_passes" > $OUT/tests.log 2>&1
timeout 300 python tools/ab_env.py SBD_CROSS_DCI=0 SBD_CROSS_DCI=1 --points cfg1 --steps 20 > $OUT/ab_dci.jsonl 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cross_kernel_dci -s 2 -c 1 -o $OUT/dci python tools/sigma_probe.py 12 6 0 2 > $OUT/ncu_dci.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/cfg1_launches.csv python tools/sigma_probe.py 12 6 0 2 > /dev/null 2>&1
for pt in "26 7 10000" "36 27 30000" "40 10 31622" "12 6 0"; do
  SBD_LIB=$PWD/paper_2601_16637_b200/_timing/libsbd_b200.so timeout 300 python -c "
import sys,time; sys.path.insert(0,'.')
from paper_2601_16637_b200 import HamiltonianApplier, SelectedBasis, synth
norb,ne,ns=[int(v) for v in '$pt'.split()]
t0=time.time(); table=synth.random_integrals(norb, seed=1)
if ns==0: basis=synth.full_product_basis(norb,ne,ne)
else:
    a,b=synth.random_product_strings(norb,ne,ne,ns,ns,seed=2); t1=time.time(); basis=SelectedBasis.product(a.tolist(),b.tolist(),norb,ne,ne)
t2=time.time(); app=HamiltonianApplier(basis,table); t3=time.time()
print('point',norb,ne,ns,'synth+basis %.3f s'%(t2-t0),'applier %.3f s'%(t3-t2), flush=True)
" >> $OUT/setup_timing.log 2>&1
done
echo done > $OUT/DONE
