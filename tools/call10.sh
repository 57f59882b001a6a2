# staged exact greedy sweep: parity (all GPU tests + the full cfg2 selection
# incl. the capped level vs the reference's own run) and timing vs the
# generic sweep (IMB_SWEEP_GENERIC=1) on cfg2 levels 0-1
A=gpurun_out/c10; mkdir -p $A
timeout 900 python -m pytest tests -m gpu -q -x > $A/pytest.log 2>&1; tail -1 $A/pytest.log
IMB_SWEEP_GENERIC=1 python tools/greedy_levels.py cfg2 2 > $A/generic.log 2>&1; cat $A/generic.log
python tools/greedy_levels.py cfg2 2 > $A/staged.log 2>&1; cat $A/staged.log
python tools/greedy_levels.py cfg4 2 > $A/staged_cfg4.log 2>&1; cat $A/staged_cfg4.log
IMB_FULL=1 timeout 1200 python -m pytest tests -m gpu -q -x -k "cfg2_full_selection" > $A/pytest_full.log 2>&1; tail -1 $A/pytest_full.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_greedy_cfg2.csv python tools/greedy_levels.py cfg2 2 > /dev/null 2>&1
for w in cfg4 cfg2; do
  timeout 600 python bench.py --workload $w --greedy-cache devcache/${w}_controls.npz --no-fast --no-cpu-baseline --steps 3 > $A/$w.json 2>/dev/null
  python -c "import json; d=json.load(open('$A/$w.json')); print('$w', round(d['value'],1), d['roofline']['frac'])"
done
timeout 600 python bench.py --workload raw --raw nc=16384,nv=10000000,R=1,D=inf --no-fast --no-cpu-baseline --steps 3 > $A/rawR1.json 2>/dev/null
python -c "import json; d=json.load(open('$A/rawR1.json')); print('rawR1', round(d['value'],1), d['roofline']['frac'])"
