cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -Xcompiler -pthread tools/micro/graph_inst.cu -o /tmp/graph_inst
echo "== exec graphs destroyed" > gpurun_out/graph_inst.log
timeout 900 /tmp/graph_inst >> gpurun_out/graph_inst.log 2>&1
echo "== exec graphs kept" >> gpurun_out/graph_inst.log
KEEP=1 timeout 900 /tmp/graph_inst >> gpurun_out/graph_inst.log 2>&1
