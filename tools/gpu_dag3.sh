cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16 HLU_PLAN_TIMING=1
timeout 900 python tools/dag_compare.py cfg3p_8192 1 2 5 10 > gpurun_out/dag3_cfg3p.log 2>&1; echo "rc $?" >> gpurun_out/dag3_cfg3p.log
timeout 1500 python tools/dag_compare.py cfg2 5 10 > gpurun_out/dag3_cfg2.log 2>&1; echo "rc $?" >> gpurun_out/dag3_cfg2.log
