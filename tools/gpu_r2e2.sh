cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/e2_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/e2_smoke.log 2>&1; echo "rc $?" >> $O/e2_smoke.log
HLU_E2E_TIMING=1 timeout 1500 python bench.py --steps 3 --warmup 3 > $O/e2_bench.json 2> $O/e2_bench.err; echo "bench rc $?" >> $O/e2_bench.err
tail -c 3000 $O/e2_bench.err > $O/e2_bench.err.tail; mv $O/e2_bench.err.tail $O/e2_bench.err
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > $O/e2_pytest.log 2>&1; echo "pytest rc $?" >> $O/e2_pytest.log
timeout 600 python tools/ncu_case.py cfg3p_8192 > $O/e2_case_cfg3p.json 2> /tmp/e2_case.err || { tail -20 /tmp/e2_case.err; echo plain failed; exit 1; }
timeout 1100 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/e2_launches.csv python tools/ncu_case.py cfg3p_8192 > /tmp/e2_ncu_launch.log 2>&1; echo launch_rc=$?
python tools/rkt_traffic.py /tmp/e2_launches.csv $O/e2_case_cfg3p.json $O/e2_launches_cfg3p_summary.txt - ; echo summary_rc=$?
gzip -c /tmp/e2_launches.csv > $O/e2_launches_cfg3p.csv.gz; ls -la $O/e2_launches_cfg3p.csv.gz
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_rkt -c 3000 --csv --log-file /tmp/e2_traffic.csv python tools/ncu_case.py cfg3p_8192 > /tmp/e2_ncu_traffic.log 2>&1; echo traffic_rc=$?
python tools/rkt_traffic.py /tmp/e2_traffic.csv $O/e2_case_cfg3p.json $O/e2_traffic_cfg3p_summary.txt $O/e2_rkt_traffic.json --partial; echo traffic_summary_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rkt_(a|b|c|r|bw)|k_gemm|k_trsm|k_getrf" -s 2000 -c 36 -o /tmp/e2_prof python tools/ncu_case.py cfg3p_8192 > /tmp/e2_ncu_full.log 2>&1; echo full_rc=$?
ncu -i /tmp/e2_prof.ncu-rep --page raw --csv > $O/e2_full_raw.csv 2>/dev/null; ls -la /tmp/e2_prof.ncu-rep $O/e2_full_raw.csv
du -sh $O
