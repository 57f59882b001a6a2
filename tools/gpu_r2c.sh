# direct gather kernel: parity, cfg3 A/B; cfg4 greedy timeline; wall-distance timings + ncu
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out devcache
cp gpurun_in/*.npz devcache/ 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_exact_tiled.py tests/test_gpu_wing.py tests/test_gpu_pipeline.py -m gpu -x -q > gpurun_out/pytest_direct.log 2>&1; echo rc=$? >> gpurun_out/pytest_direct.log
tail -n 6 gpurun_out/pytest_direct.log
for v in default n4 tile; do
  IMB_GATHER=$v IMB_COUNT_PAIRS= timeout 900 python bench.py --workload cfg3 --greedy-cache devcache/cfg3_controls.npz --steps 5 --no-deform --no-cpu-baseline --no-fast > gpurun_out/bench_cfg3_$v.json 2> gpurun_out/bench_cfg3_$v.err
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_cfg3_*.json")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["value"], d["roofline"]["frac"], d.get("kernel_ms_avg"), d.get("hbm_passes"))
PY
for c in cfg2 cfg3 cfg4; do timeout 600 python tools/hbm_passes.py $c 1.0 1.0 3 > gpurun_out/hbm_$c.json 2> gpurun_out/hbm_$c.err; cat gpurun_out/hbm_$c.json; done
# cfg4 greedy with the per-step timeline
IMB_SPEC_LOG=gpurun_out/spec_cfg4.log timeout 900 python bench.py --workload cfg4 --greedy-cache devcache/cfg4_controls.npz --steps 2 --no-deform --no-cpu-baseline --no-fast > gpurun_out/bench_cfg4_spec.json 2> gpurun_out/bench_cfg4_spec.err
tail -3 gpurun_out/bench_cfg4_spec.err
cp devcache/cfg4_controls.npz gpurun_out/ 2>/dev/null
gzip -f gpurun_out/spec_cfg4.log
# ncu: wall distance + compaction on cfg3 (after the same command ran plain above)
timeout 600 python tools/hbm_passes.py cfg3 1.0 1.0 1 > gpurun_out/hbm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_wall_distance|k_count_active|k_scan_counts|k_scatter_active" -c 8 -o gpurun_out/ncu_hbm_cfg3 -f python tools/hbm_passes.py cfg3 1.0 1.0 1 > gpurun_out/ncu_hbm.log 2>&1; echo ncu rc=$?
ls -la gpurun_out | head -50
