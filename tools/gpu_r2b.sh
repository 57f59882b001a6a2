# power-of-two-R pre-scaling: parity tests, then cfg2 / cfg3 exact A/B
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out devcache
timeout 900 python -m pytest tests/test_gpu_exact_tiled.py tests/test_gpu_wing.py tests/test_gpu_pipeline.py -m gpu -x -q > gpurun_out/pytest_pre.log 2>&1; echo rc=$? >> gpurun_out/pytest_pre.log
tail -n 6 gpurun_out/pytest_pre.log
for c in cfg2 cfg3; do
  timeout 900 python bench.py --workload $c --greedy-cache devcache/${c}_controls.npz --steps 5 --no-deform --no-cpu-baseline --no-fast > gpurun_out/bench_${c}_pre.json 2> gpurun_out/bench_${c}_pre.err
  IMB_NO_PRESCALE=1 timeout 900 python bench.py --workload $c --greedy-cache devcache/${c}_controls.npz --steps 5 --no-deform --no-cpu-baseline --no-fast > gpurun_out/bench_${c}_nopre.json 2> gpurun_out/bench_${c}_nopre.err
  IMB_COUNT_PAIRS=1 timeout 900 python bench.py --workload $c --greedy-cache devcache/${c}_controls.npz --steps 2 --no-deform --no-cpu-baseline --no-fast > gpurun_out/bench_${c}_count.json 2> gpurun_out/bench_${c}_count.err
done
cp devcache/*.npz gpurun_out/ 2>/dev/null
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_cfg*_*.json")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["value"], d["roofline"]["frac"], d.get("kernel_ms_avg"), d.get("pairs_evaluated"), d.get("greedy_seconds_per_level"))
PY
