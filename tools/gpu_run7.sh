cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "wide" > gpurun_out/pytest_r2g_wide.log 2>&1; echo "rc $?" >> gpurun_out/pytest_r2g_wide.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sphere_2048_l64 or cfg3p_8192 or cfg4p or cfg2" > gpurun_out/pytest_r2g.log 2>&1; echo "rc $?" >> gpurun_out/pytest_r2g.log
timeout 900 python -m pytest tests/test_gpu_assembly.py -q > gpurun_out/pytest_r2g_asm.log 2>&1; echo "rc $?" >> gpurun_out/pytest_r2g_asm.log
