cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm|k_getrf|k_trsm" -o /tmp/e8_prof python tools/kernel_roofline.py > /tmp/e8_ncu.log 2>&1; echo "ncu rc $?" >> $O/e8_rc.txt
ncu -i /tmp/e8_prof.ncu-rep --page raw --csv > $O/e8_full_raw.csv 2>/dev/null
ncu -i /tmp/e8_prof.ncu-rep --page details -k regex:"k_trsm" > /tmp/e8_details.txt 2>/dev/null; head -230 /tmp/e8_details.txt > $O/e8_details_trsm.txt
ncu -i /tmp/e8_prof.ncu-rep --page source --csv -k regex:k_trsm --print-source sass > /tmp/e8_trsm_src.csv 2>/dev/null; gzip -c /tmp/e8_trsm_src.csv > $O/e8_trsm_src.csv.gz
du -sh $O
