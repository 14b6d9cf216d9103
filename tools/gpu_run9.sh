cd $GRAFT_REPO_ROOT
export HLU_PRODUCT_PAIR_MAX=128
for i in 1 2; do
timeout 600 python tools/diag_wide.py sphere_2048_l64 > gpurun_out/diag_wide_a$i.log 2>&1
HLU_RKT_SERIAL=1 timeout 600 python tools/diag_wide.py sphere_2048_l64 > gpurun_out/diag_wide_s$i.log 2>&1
HLU_RKT_SERIAL=1 HLU_CHAINS=0 HLU_NOGRAPH=1 timeout 600 python tools/diag_wide.py sphere_2048_l64 > gpurun_out/diag_wide_n$i.log 2>&1
done
