cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_matvec.py tests/test_gpu_assembly.py -m gpu -q -x -k "not cfg3 and not cfg2" > $O/e14_pytest_quick.log 2>&1; echo "pytest quick rc $?" >> $O/e14_rc.txt
timeout 300 python tools/kernel_roofline.py > $O/e14_kernels.jsonl 2> /tmp/e14_k.err; echo "kernels rc $?" >> $O/e14_rc.txt; tail -3 /tmp/e14_k.err >> $O/e14_rc.txt
HLU_PLAN_TIMING=1 timeout 600 python tools/dag_compare.py cfg2 5 2>&1 | grep "schedule: dag\|cfg2" > $O/e14_cfg2.log
HLU_PLAN_TIMING=1 timeout 600 python tools/dag_compare.py cfg3p_8192 5 2>&1 | grep "cfg3p" > $O/e14_cfg3p.log
