cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16
timeout 900 python tools/dag_timeline.py cfg3p_8192 5 > gpurun_out/dag4_tl_cfg3p.log 2>&1; echo "rc $?" >> gpurun_out/dag4_tl_cfg3p.log
timeout 1500 python tools/dag_timeline.py cfg2 10 > gpurun_out/dag4_tl_cfg2.log 2>&1; echo "rc $?" >> gpurun_out/dag4_tl_cfg2.log
