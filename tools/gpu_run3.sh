cd $GRAFT_REPO_ROOT
timeout 600 python -X faulthandler -m pytest tests/test_gpu_parity.py -x -q -k "lu_ or trsm or gemm or eps0 or known" > gpurun_out/pytest_r2c_unit.log 2>&1; echo "rc $?" >> gpurun_out/pytest_r2c_unit.log
timeout 900 python -X faulthandler bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err; echo "bench rc $?" >> gpurun_out/bench_r2c.err
