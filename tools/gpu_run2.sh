# GPU session script: tests, fp64 peak microbenchmark, bench, ncu of k_gemm
cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/micro/fp64_peak.cu -o /tmp/fp64_peak && /tmp/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2b.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_r2b.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo "bench rc $?" >> gpurun_out/bench_r2b.err
