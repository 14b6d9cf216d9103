cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "wide_dense_product_bem" > gpurun_out/pytest_r2h.log 2>&1; echo "rc $?" >> gpurun_out/pytest_r2h.log
