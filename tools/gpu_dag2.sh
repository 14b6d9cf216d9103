cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16
timeout 2400 python tools/dag_compare.py cfg3 20 10 > gpurun_out/dag2_cfg3.log 2>&1; echo "rc $?" >> gpurun_out/dag2_cfg3.log
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/dag2_cfg3.log
