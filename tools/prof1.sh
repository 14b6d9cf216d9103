set -x
timeout 600 python tools/run_case_nograph.py cfg3p_8192 > gpurun_out/plain_cfg3p.log 2>&1 || { echo plain failed; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3p.csv python tools/run_case_nograph.py cfg3p_8192 > gpurun_out/ncu_launch.log 2>&1; echo launch_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rkt_(a|b|c|r|bw)|k_gemm" -s 700 -c 12 -o gpurun_out/prof_cfg3p python tools/run_case_nograph.py cfg3p_8192 > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
