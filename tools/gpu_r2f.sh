# div2 (cfg4 headline), balanced sweep tiles: parity, cfg4 exact A/B, k_sweep ncu
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out devcache
cp gpurun_in/*.npz devcache/ 2>/dev/null
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/pytest_all.log
tail -n 6 gpurun_out/pytest_all.log
timeout 600 python tools/greedy_levels.py cfg3 1 > gpurun_out/greedy_cfg3.log 2>&1; tail -1 gpurun_out/greedy_cfg3.log
# cfg4 volume kernel with fixed controls from the cache when present, else 2 levels of device greedy
timeout 1500 python bench.py --workload cfg4 --greedy-cache devcache/cfg4_controls.npz --steps 5 --no-deform --no-cpu-baseline --no-fast > gpurun_out/bench_cfg4_div2.json 2> gpurun_out/bench_cfg4_div2.err
IMB_NO_DIV2=1 timeout 1500 python bench.py --workload cfg4 --greedy-cache devcache/cfg4_controls.npz --steps 5 --no-deform --no-cpu-baseline --no-fast > gpurun_out/bench_cfg4_nodiv2.json 2> gpurun_out/bench_cfg4_nodiv2.err
cp devcache/cfg4_controls.npz gpurun_out/ 2>/dev/null
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_cfg4_*.json")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["value"], d["roofline"]["frac"], d.get("kernel_ms_avg"), d.get("greedy_seconds_per_level"))
PY
IMB_SPEC=0 timeout 600 python tools/greedy_levels.py cfg2 2 > gpurun_out/greedy_cfg2_seq.log 2>&1 && \
IMB_SPEC=0 ncu --set full --clock-control none --import-source on -k regex:"k_sweep" --launch-skip 1200 -c 1 -o /tmp/sw -f python tools/greedy_levels.py cfg2 2 > gpurun_out/ncu_sw.log 2>&1
ncu -i /tmp/sw.ncu-rep --page raw --csv > gpurun_out/ncu_k_sweep_cfg2_raw.csv 2>/dev/null
ncu -i /tmp/sw.ncu-rep --page details --csv > gpurun_out/ncu_k_sweep_cfg2_details.csv 2>/dev/null
du -sh gpurun_out
