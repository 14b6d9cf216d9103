cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1
timeout 300 python -X faulthandler -m pytest tests/test_gpu_parity.py -x -q -k "eps0 or mixed_192" > gpurun_out/pytest_r2d.log 2>&1; echo "rc $?" >> gpurun_out/pytest_r2d.log
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -X faulthandler -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2d.log 2>&1; echo "rc $?" >> gpurun_out/smoke_r2d.log
HLU_CHAINS=0 timeout 300 python -X faulthandler -m pytest tests/test_gpu_parity.py -x -q -k "sphere_1024" > gpurun_out/pytest_r2d_nochain.log 2>&1; echo "rc $?" >> gpurun_out/pytest_r2d_nochain.log
