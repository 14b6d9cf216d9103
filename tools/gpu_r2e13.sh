cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16
O=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/e13_smoke.log 2>&1; echo "smoke rc $?" >> $O/e13_rc.txt
timeout 3000 python -m pytest tests -m gpu -q -x --durations=10 > $O/e13_pytest.log 2>&1; echo "pytest rc $?" >> $O/e13_rc.txt
( time HLU_E2E_TIMING=1 timeout 1500 python bench.py > $O/e13_bench.json 2> /tmp/e13_bench.err ) 2> $O/e13_bench_time.txt; echo "bench rc $?" >> $O/e13_rc.txt; tail -c 2500 /tmp/e13_bench.err > $O/e13_bench.err
( time timeout 600 python bench.py --impl reference > $O/e13_bench_ref.json 2> /tmp/e13_ref.err ) 2> $O/e13_ref_time.txt; echo "ref rc $?" >> $O/e13_rc.txt
for cfg in cfg1 cfg2 cfg4p cfg5s cfg5; do
  timeout 1200 python bench.py --config $cfg --steps 3 --warmup 3 --no-kernel-roofline --no-cpu-baseline > $O/e13_$cfg.json 2> /tmp/e13_$cfg.err; echo "$cfg rc $?" >> $O/e13_rc.txt
done
timeout 1500 python tools/dag_timeline.py cfg3 5 > $O/e13_timeline_cfg3_5us.txt 2>&1; echo "timeline rc $?" >> $O/e13_rc.txt
rm -f $O/timeline_*.npz
du -sh $O
