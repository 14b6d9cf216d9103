cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 600 python tools/dag_compare.py sphere_2048_l64 20 > gpurun_out/dag1_small.log 2>&1; echo "rc $?" >> gpurun_out/dag1_small.log
timeout 900 python tools/dag_compare.py cfg3p_8192 10 20 50 > gpurun_out/dag1_cfg3p.log 2>&1; echo "rc $?" >> gpurun_out/dag1_cfg3p.log
timeout 1500 python tools/dag_compare.py cfg2 20 50 > gpurun_out/dag1_cfg2.log 2>&1; echo "rc $?" >> gpurun_out/dag1_cfg2.log
