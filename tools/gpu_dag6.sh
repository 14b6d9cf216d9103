cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16 HLU_FUSE_MAX=0
for pr in off 200,2000 50,500 500,5000 0,100; do
echo "== prio $pr" >> gpurun_out/dag6_cfg3p.log
HLU_DAG_PRIO=$pr timeout 900 python tools/dag_compare.py cfg3p_8192 5 2>&1 | grep -v "^build" >> gpurun_out/dag6_cfg3p.log
done
for pr in off 200,2000; do
echo "== prio $pr" >> gpurun_out/dag6_cfg2.log
HLU_DAG_PRIO=$pr timeout 1500 python tools/dag_compare.py cfg2 5 2>&1 | grep -v "^build" >> gpurun_out/dag6_cfg2.log
done
HLU_DAG_PRIO=200,2000 timeout 900 python tools/dag_timeline.py cfg3p_8192 5 > gpurun_out/dag6_tl_cfg3p.log 2>&1
