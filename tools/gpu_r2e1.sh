cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/e1_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e1_smoke.log 2>&1; echo "rc $?" >> gpurun_out/e1_smoke.log
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/e1_bench.json 2> gpurun_out/e1_bench.err; echo "bench rc $?" >> gpurun_out/e1_bench.err
timeout 600 python tools/ncu_case.py cfg3p_8192 > gpurun_out/e1_case_cfg3p.json 2> gpurun_out/e1_case_cfg3p.err || { echo plain failed; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/e1_launches_cfg3p.csv python tools/ncu_case.py cfg3p_8192 > gpurun_out/e1_ncu_launch.log 2>&1; echo launch_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_rkt_(a|b|c|r|bw|w)|k_gemm|k_trsm|k_getrf" -s 2000 -c 40 -o gpurun_out/e1_prof_cfg3p python tools/ncu_case.py cfg3p_8192 > gpurun_out/e1_ncu_full.log 2>&1; echo full_rc=$?
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/e1_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/e1_pytest.log
