cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p1_smoke.log 2>&1; echo "rc $?" >> gpurun_out/p1_smoke.log
timeout 3000 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/p1_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/p1_pytest.log
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/p1_bench.json 2> gpurun_out/p1_bench.err; echo "bench rc $?" >> gpurun_out/p1_bench.err
