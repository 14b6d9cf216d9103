cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1 HLU_ASSEMBLY_WORKERS=16
O=gpurun_out
run() { # name, env..., -- args
  name=$1; shift
  timeout 1500 env "$@" > $O/e3_$name.json 2> /tmp/e3_$name.err; echo "$name rc $?" >> $O/e3_rc.txt; tail -c 1500 /tmp/e3_$name.err > $O/e3_$name.err
}
run cfg3_slot5 HLU_DAG_SLOT_US=5 HLU_E2E_TIMING=1 python bench.py --steps 3 --warmup 3 --no-kernel-roofline --no-cpu-baseline
run cfg2 python bench.py --config cfg2 --steps 3 --warmup 3 --no-kernel-roofline --no-cpu-baseline
run cfg1 python bench.py --config cfg1 --steps 5 --warmup 3 --no-kernel-roofline --no-cpu-baseline
run cfg4p python bench.py --config cfg4p --steps 3 --warmup 3 --no-kernel-roofline --no-cpu-baseline
run cfg5s python bench.py --config cfg5s --steps 3 --warmup 3 --no-kernel-roofline --no-cpu-baseline
run cfg5 python bench.py --config cfg5 --steps 3 --warmup 3 --no-kernel-roofline --no-cpu-baseline
timeout 900 python tools/dag_timeline.py cfg2 10 > $O/e3_timeline_cfg2_10us.txt 2>&1; echo "timeline cfg2 rc $?" >> $O/e3_rc.txt
timeout 1200 python tools/dag_timeline.py cfg3 20 > $O/e3_timeline_cfg3_20us.txt 2>&1; echo "timeline cfg3 rc $?" >> $O/e3_rc.txt
rm -f $O/timeline_*.npz
du -sh $O
