cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "trsm or gemm or lu_ or factorization_parity or solve_parity or dag_schedule" > $O/e6_pytest_quick.log 2>&1; echo "pytest quick rc $?" >> $O/e6_rc.txt
timeout 300 python tools/kernel_roofline.py > $O/e6_kernels.jsonl 2> /tmp/e6_k.err; echo "kernels rc $?" >> $O/e6_rc.txt; tail -3 /tmp/e6_k.err >> $O/e6_rc.txt
HLU_PLAN_TIMING=1 timeout 600 python tools/dag_compare.py cfg2 5 2>&1 | grep "schedule: dag\|cfg2" > $O/e6_cfg2.log
HLU_PLAN_TIMING=1 timeout 600 python tools/dag_compare.py cfg3p_8192 5 2>&1 | grep "cfg3p" > $O/e6_cfg3p.log
