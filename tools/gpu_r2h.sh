export PYTHONUNBUFFERED=1
A=gpurun_out/art2; mkdir -p $A devcache; cp gpurun_in/*.npz devcache/ 2>/dev/null
timeout 2400 python -m pytest tests -m gpu -x -q > $A/pytest_gpu.log 2>&1; tail -1 $A/pytest_gpu.log
for c in cfg2 cfg3 cfg4; do timeout 600 python tools/hbm_passes.py $c 1.0 1.0 5 > $A/hbm_$c.json 2> $A/hbm_$c.err; cat $A/hbm_$c.json; done
python tools/hbm_passes.py cfg3 1.0 1.0 1 > $A/hbm_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_count_active|k_scan_counts|k_scatter_active" -c 6 -o /tmp/cp -f python tools/hbm_passes.py cfg3 1.0 1.0 1 > $A/ncu_cp.log 2>&1
ncu -i /tmp/cp.ncu-rep --page raw --csv > $A/ncu_compaction_cfg3_raw.csv 2>/dev/null
ncu -i /tmp/cp.ncu-rep --page details --csv > $A/ncu_compaction_cfg3_details.csv 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_hbm_passes_cfg3.csv python tools/hbm_passes.py cfg3 1.0 1.0 1 > /dev/null 2>&1
( time python bench.py > $A/bench_cfg4.json 2> $A/bench_cfg4.err ) 2> $A/bench_cfg4.time; tail -3 $A/bench_cfg4.time
for c in cfg2 cfg3; do
  python bench.py --workload $c --greedy-cache devcache/${c}_controls.npz --steps 5 > $A/bench_$c.json 2> $A/bench_$c.err
done
du -sh gpurun_out
