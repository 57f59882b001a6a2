# Round-end measurement set (run on the GPU box):
#   default bench (no cache), pytest -m gpu log, launch list of the default
#   bench under ncu (per-launch times), one ncu --set full capture of the top
#   kernel exported to CSV (raw + source), cfg3 / cfg4 bench lines.
set -x
mkdir -p gpurun_out/art
python -m pytest tests -m gpu -q > gpurun_out/art/pytest_gpu.log 2>&1; tail -1 gpurun_out/art/pytest_gpu.log
python bench.py > gpurun_out/art/bench_cfg2.json 2> gpurun_out/art/bench_cfg2.err
python bench.py --impl reference > gpurun_out/art/bench_reference.json 2> gpurun_out/art/bench_reference.err
for c in cfg3 cfg4; do
  python bench.py --workload $c --greedy-cache devcache/${c}_controls.npz --steps 5 > gpurun_out/art/bench_$c.json 2> gpurun_out/art/bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/art/launches_cfg2.csv \
    python bench.py --greedy-cache devcache/cfg2_controls.npz --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_volume_exact_tiled --launch-skip 8 -c 1 \
    -o /tmp/k_exact python bench.py --greedy-cache devcache/cfg2_controls.npz --steps 2 --warmup 3 --no-cpu-baseline --no-fast > /dev/null 2>&1
ncu -i /tmp/k_exact.ncu-rep --page raw --csv > gpurun_out/art/ncu_exact_cfg2_raw.csv 2>/dev/null
ncu -i /tmp/k_exact.ncu-rep --page details --csv > gpurun_out/art/ncu_exact_cfg2_details.csv 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:k_volume_fast --launch-skip 2 -c 1 \
    -o /tmp/k_fast python bench.py --workload cfg4 --greedy-cache devcache/cfg4_controls.npz --precision fp64 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu -i /tmp/k_fast.ncu-rep --page raw --csv > gpurun_out/art/ncu_fast_cfg4_raw.csv 2>/dev/null
ncu -i /tmp/k_fast.ncu-rep --page details --csv > gpurun_out/art/ncu_fast_cfg4_details.csv 2>/dev/null
ls -la gpurun_out/art
