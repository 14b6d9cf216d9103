cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16
O=gpurun_out
HLU_DAG_SLOT_US=5 HLU_E2E_TIMING=1 timeout 1500 python bench.py --steps 3 --warmup 3 > $O/e4_bench_slot5.json 2> /tmp/e4_bench.err; echo "bench slot5 rc $?" >> $O/e4_rc.txt; tail -c 2500 /tmp/e4_bench.err > $O/e4_bench_slot5.err
export HLU_PLAN_TIMING=1
timeout 600 python tools/dag_compare.py cfg2 5 2>&1 | grep "schedule: dag\|cfg2" > $O/e4_inst_default.log
HLU_DAG_PRIO=off timeout 600 python tools/dag_compare.py cfg2 5 2>&1 | grep "schedule: dag\|cfg2" > $O/e4_inst_prio_off.log
HLU_DAG_CHUNK_NODES=3000 timeout 600 python tools/dag_compare.py cfg2 5 2>&1 | grep "schedule: dag\|cfg2" > $O/e4_inst_chunk3k.log
HLU_DAG_CHUNK_NODES=48000 timeout 600 python tools/dag_compare.py cfg2 5 2>&1 | grep "schedule: dag\|cfg2" > $O/e4_inst_chunk48k.log
du -sh $O
HLU_DAG_JOIN=1 timeout 600 python tools/dag_compare.py cfg2 5 2>&1 | grep "schedule: dag\|cfg2" > $O/e4_inst_join.log
HLU_DAG_JOIN=1 HLU_DAG_PRIO=off timeout 600 python tools/dag_compare.py cfg2 5 2>&1 | grep "schedule: dag\|cfg2" > $O/e4_inst_join_prio_off.log
