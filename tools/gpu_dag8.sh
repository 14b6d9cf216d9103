cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16 HLU_PLAN_TIMING=1
timeout 1500 python tools/dag_compare.py cfg2 5 2>&1 | grep "schedule: dag\|cfg2" > gpurun_out/dag8_cfg2.log
HLU_DAG_PRIO=off timeout 1500 python tools/dag_compare.py cfg2 5 2>&1 | grep "schedule: dag\|cfg2" >> gpurun_out/dag8_cfg2.log
