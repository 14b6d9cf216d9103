cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16
O=gpurun_out
for pr in "200,2000" "50,500" "1000,10000" "20,200" "off"; do
  echo "== HLU_DAG_PRIO=$pr" >> $O/e15_prio.log
  HLU_DAG_PRIO=$pr timeout 600 python tools/dag_compare.py cfg2 5 2>&1 | grep "cfg2 dag" >> $O/e15_prio.log
done
timeout 600 python tools/ncu_case.py cfg3p_8192 > $O/e15_case_cfg3p.json 2> /tmp/e15_case.err || { tail -20 /tmp/e15_case.err; echo plain failed; exit 1; }
timeout 1100 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/e15_launches.csv python tools/ncu_case.py cfg3p_8192 > /tmp/e15_ncu_launch.log 2>&1; echo launch_rc=$? >> $O/e15_rc.txt
python tools/rkt_traffic.py /tmp/e15_launches.csv $O/e15_case_cfg3p.json $O/e15_launches_cfg3p_summary.txt - ; echo summary_rc=$? >> $O/e15_rc.txt
gzip -c /tmp/e15_launches.csv > $O/e15_launches_cfg3p.csv.gz
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_rkt -c 3000 --csv --log-file /tmp/e15_traffic.csv python tools/ncu_case.py cfg3p_8192 > /tmp/e15_ncu_traffic.log 2>&1; echo traffic_rc=$? >> $O/e15_rc.txt
python tools/rkt_traffic.py /tmp/e15_traffic.csv $O/e15_case_cfg3p.json $O/e15_traffic_cfg3p_summary.txt $O/e15_rkt_traffic.json --partial; echo traffic_summary_rc=$? >> $O/e15_rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rkt_(a|b|c|r|bw)|k_gemm|k_trsm|k_getrf" -s 2000 -c 36 -o /tmp/e15_prof python tools/ncu_case.py cfg3p_8192 > /tmp/e15_ncu_full.log 2>&1; echo full_rc=$? >> $O/e15_rc.txt
ncu -i /tmp/e15_prof.ncu-rep --page raw --csv > $O/e15_full_raw.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:"k_gemm|k_getrf|k_trsm|k_rkt" -o /tmp/e15_alone python tools/kernel_roofline.py > /tmp/e15_alone.log 2>&1; echo alone_rc=$? >> $O/e15_rc.txt
ncu -i /tmp/e15_alone.ncu-rep --page raw --csv > $O/e15_alone_raw.csv 2>/dev/null
du -sh $O
