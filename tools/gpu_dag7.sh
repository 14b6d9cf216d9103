cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16 HLU_PLAN_TIMING=1
timeout 900 python tools/dag_compare.py cfg3p_8192 5 2>&1 | grep -v "^build\|^plan:" > gpurun_out/dag7_cfg3p.log
HLU_DAG_CHUNK_NODES=4000 timeout 900 python tools/dag_compare.py cfg3p_8192 5 2>&1 | grep -v "^build\|^plan:" >> gpurun_out/dag7_cfg3p.log
HLU_DAG_CHUNK_NODES=30000 timeout 900 python tools/dag_compare.py cfg3p_8192 5 2>&1 | grep -v "^build\|^plan:" >> gpurun_out/dag7_cfg3p.log
timeout 1500 python tools/dag_compare.py cfg2 5 2>&1 | grep -v "^build\|^plan:" > gpurun_out/dag7_cfg2.log
timeout 2400 python tools/dag_compare.py cfg3 10 5 2>&1 | grep -v "^build\|^plan:" > gpurun_out/dag7_cfg3.log
