cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/micro/fp64_peak.cu -o /tmp/fp64_peak && /tmp/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s2a.log 2>&1; echo "rc $?" >> gpurun_out/smoke_s2a.log
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=30 > gpurun_out/pytest_s2a.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_s2a.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_s2a.json 2> gpurun_out/bench_s2a.err; echo "bench rc $?" >> gpurun_out/bench_s2a.err
