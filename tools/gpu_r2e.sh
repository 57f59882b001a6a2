# 8-warp sweeps, stack-light wall distance, 64-thread gather CTAs: full suite, timings, ncu
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out devcache
cp gpurun_in/*.npz devcache/ 2>/dev/null
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/pytest_all.log
tail -n 6 gpurun_out/pytest_all.log
timeout 600 python tools/greedy_levels.py cfg2 3 > gpurun_out/greedy_cfg2.log 2>&1; tail -1 gpurun_out/greedy_cfg2.log
timeout 600 python tools/greedy_levels.py cfg3 1 > gpurun_out/greedy_cfg3.log 2>&1; tail -1 gpurun_out/greedy_cfg3.log
IMB_SPEC_LOG=/tmp/spec_cfg4.log timeout 900 python tools/greedy_levels.py cfg4 2 > gpurun_out/greedy_cfg4.log 2>&1; tail -2 gpurun_out/greedy_cfg4.log
python tools/spec_timeline.py /tmp/spec_cfg4.log > gpurun_out/spec_timeline_cfg4.txt 2>&1; tail -6 gpurun_out/spec_timeline_cfg4.txt
for c in cfg2 cfg3 cfg4; do timeout 600 python tools/hbm_passes.py $c 1.0 1.0 5 > gpurun_out/hbm_$c.json 2> gpurun_out/hbm_$c.err; cat gpurun_out/hbm_$c.json; done
for v in default t256; do
  IMB_GATHER=$v timeout 900 python bench.py --workload cfg3 --greedy-cache devcache/cfg3_controls.npz --steps 5 --no-deform --no-cpu-baseline --no-fast > gpurun_out/bench_cfg3_$v.json 2> gpurun_out/bench_cfg3_$v.err
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_cfg3_*.json")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["value"], d["roofline"]["frac"], d.get("kernel_ms_avg"))
PY
IMB_SPEC=0 timeout 600 python tools/greedy_levels.py cfg2 2 > gpurun_out/greedy_cfg2_seq.log 2>&1 && \
IMB_SPEC=0 ncu --set full --clock-control none --import-source on -k regex:"k_sweep" --launch-skip 1200 -c 1 -o /tmp/sw -f python tools/greedy_levels.py cfg2 2 > gpurun_out/ncu_sw.log 2>&1
ncu -i /tmp/sw.ncu-rep --page raw --csv > gpurun_out/ncu_k_sweep_cfg2_raw.csv 2>/dev/null
ncu -i /tmp/sw.ncu-rep --page details --csv > gpurun_out/ncu_k_sweep_cfg2_details.csv 2>/dev/null
ncu -i /tmp/sw.ncu-rep --page source --csv > gpurun_out/ncu_k_sweep_cfg2_source.csv 2>/dev/null
timeout 600 python tools/hbm_passes.py cfg3 1.0 1.0 1 > gpurun_out/hbm_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_hbm_cfg3.csv python tools/hbm_passes.py cfg3 1.0 1.0 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"k_wall_distance|k_count_active|k_scan_counts|k_scatter_active" -c 4 -o /tmp/wd -f python tools/hbm_passes.py cfg3 1.0 1.0 1 > gpurun_out/ncu_wd.log 2>&1
ncu -i /tmp/wd.ncu-rep --page raw --csv > gpurun_out/ncu_hbm_passes_cfg3_raw.csv 2>/dev/null
ncu -i /tmp/wd.ncu-rep --page details --csv > gpurun_out/ncu_hbm_passes_cfg3_details.csv 2>/dev/null
timeout 600 python bench.py --workload cfg3 --greedy-cache devcache/cfg3_controls.npz --steps 1 --warmup 1 --no-deform --no-cpu-baseline --no-fast > gpurun_out/bench_cfg3_plain.json 2>&1 && \
ncu --set full --clock-control none -k regex:"k_volume_exact_direct" --launch-skip 2 -c 1 -o /tmp/gd -f python bench.py --workload cfg3 --greedy-cache devcache/cfg3_controls.npz --steps 1 --warmup 1 --no-deform --no-cpu-baseline --no-fast > gpurun_out/ncu_gd.log 2>&1
ncu -i /tmp/gd.ncu-rep --page raw --csv > gpurun_out/ncu_k_volume_exact_direct_cfg3_raw.csv 2>/dev/null
ncu -i /tmp/gd.ncu-rep --page details --csv > gpurun_out/ncu_k_volume_exact_direct_cfg3_details.csv 2>/dev/null
du -sh gpurun_out
