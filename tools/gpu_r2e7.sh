cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16
O=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/e7_smoke.log 2>&1; echo "smoke rc $?" >> $O/e7_rc.txt
HLU_PLAN_TIMING=1 timeout 600 python tools/dag_compare.py cfg2 5 2>&1 | grep "schedule: dag\|cfg2" > $O/e7_cfg2.log
timeout 3000 python -m pytest tests -m gpu -q -x --durations=10 > $O/e7_pytest.log 2>&1; echo "pytest rc $?" >> $O/e7_rc.txt
( time HLU_E2E_TIMING=1 timeout 1500 python bench.py > $O/e7_bench.json 2> /tmp/e7_bench.err ) 2> $O/e7_bench_time.txt; echo "bench rc $?" >> $O/e7_rc.txt; tail -c 2500 /tmp/e7_bench.err > $O/e7_bench.err
( time timeout 600 python bench.py --impl reference > $O/e7_bench_ref.json 2> /tmp/e7_ref.err ) 2> $O/e7_ref_time.txt; echo "ref rc $?" >> $O/e7_rc.txt; tail -c 800 /tmp/e7_ref.err > $O/e7_ref.err
