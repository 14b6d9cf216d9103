cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16
O=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/e16_smoke.log 2>&1; echo "smoke rc $?" >> $O/e16_rc.txt
timeout 3000 python -m pytest tests -m gpu -q -x --durations=5 > $O/e16_pytest.log 2>&1; echo "pytest rc $?" >> $O/e16_rc.txt
( time timeout 1500 python bench.py > $O/e16_bench.json 2> /tmp/e16_bench.err ) 2> $O/e16_bench_time.txt; echo "bench rc $?" >> $O/e16_rc.txt; tail -c 1500 /tmp/e16_bench.err > $O/e16_bench.err
