cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1
O=gpurun_out
timeout 300 python tools/kernel_roofline.py > $O/e5_kernels.jsonl 2> /tmp/e5_k.err; echo "plain rc $?" >> $O/e5_rc.txt; tail -5 /tmp/e5_k.err >> $O/e5_rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm|k_getrf|k_trsm|k_rkt" -o /tmp/e5_prof python tools/kernel_roofline.py > /tmp/e5_ncu.log 2>&1; echo "ncu rc $?" >> $O/e5_rc.txt
ncu -i /tmp/e5_prof.ncu-rep --page raw --csv > $O/e5_full_raw.csv 2>/dev/null
ncu -i /tmp/e5_prof.ncu-rep --page source --csv -k regex:k_gemm --print-source sass > /tmp/e5_gemm_src.csv 2>/dev/null; gzip -c /tmp/e5_gemm_src.csv > $O/e5_gemm_src.csv.gz
ncu -i /tmp/e5_prof.ncu-rep --page details -k regex:"k_gemm|k_rkt_r|k_trsm|k_getrf" > /tmp/e5_details.txt 2>/dev/null; gzip -c /tmp/e5_details.txt > $O/e5_details.txt.gz
ls -la /tmp/e5_prof.ncu-rep $O; du -sh $O
