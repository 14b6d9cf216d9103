cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16
timeout 600 python tools/dag_compare.py sphere_2048_l64 5 > gpurun_out/dag5_small.log 2>&1; echo "rc $?" >> gpurun_out/dag5_small.log
timeout 600 python tools/dag_compare.py mixed_192 5 >> gpurun_out/dag5_small.log 2>&1; echo "rc $?" >> gpurun_out/dag5_small.log
timeout 600 python tools/dag_compare.py cfg1 5 >> gpurun_out/dag5_small.log 2>&1; echo "rc $?" >> gpurun_out/dag5_small.log
timeout 900 python tools/dag_compare.py cfg3p_8192 2 5 10 > gpurun_out/dag5_cfg3p.log 2>&1; echo "rc $?" >> gpurun_out/dag5_cfg3p.log
HLU_FUSE_MAX=16 timeout 900 python tools/dag_compare.py cfg3p_8192 5 > gpurun_out/dag5_cfg3p_f16.log 2>&1
HLU_FUSE_MAX=256 timeout 900 python tools/dag_compare.py cfg3p_8192 5 > gpurun_out/dag5_cfg3p_f256.log 2>&1
timeout 1500 python tools/dag_compare.py cfg2 5 10 > gpurun_out/dag5_cfg2.log 2>&1; echo "rc $?" >> gpurun_out/dag5_cfg2.log
timeout 900 python tools/dag_timeline.py cfg3p_8192 5 > gpurun_out/dag5_tl_cfg3p.log 2>&1; echo "rc $?" >> gpurun_out/dag5_tl_cfg3p.log
