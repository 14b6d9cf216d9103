cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2e.log 2>&1; echo "rc $?" >> gpurun_out/smoke_r2e.log
timeout 1800 python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_r2e.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_r2e.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r2e.json 2> gpurun_out/bench_r2e.err; echo "bench rc $?" >> gpurun_out/bench_r2e.err
