cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "wide or eps0 or sharded or lu_ or trsm or gemm" > gpurun_out/pytest_r2f_unit.log 2>&1; echo "rc $?" >> gpurun_out/pytest_r2f_unit.log
timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_r2f.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_r2f.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2f.json 2> gpurun_out/bench_r2f.err; echo "bench rc $?" >> gpurun_out/bench_r2f.err
