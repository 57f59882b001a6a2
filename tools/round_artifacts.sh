# Round-end measurement set (run on the GPU box; devcache/ holds the exact
# greedy selections of cfg2/3/4 from an earlier device run, bench.py
# --greedy-cache):
#   default bench (no cache: greedy on the device in setup), pytest -m gpu,
#   smoke, reference arm, cfg3 / cfg4 lines, raw-sweep cells (FP64 / FP32),
#   launch list of the default bench under ncu (per-launch times), one
#   ncu --set full capture per volume kernel (exact / fast / FP32), exported
#   to CSV (raw + details).
set -x
A=gpurun_out/art
mkdir -p $A
python -m pytest tests -m gpu -q > $A/pytest_gpu.log 2>&1; tail -1 $A/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $A/smoke.log 2>&1; tail -1 $A/smoke.log
python bench.py > $A/bench_cfg2.json 2> $A/bench_cfg2.err
python bench.py --impl reference > $A/bench_reference.json 2> $A/bench_reference.err
for c in cfg3 cfg4; do
  python bench.py --workload $c --greedy-cache devcache/${c}_controls.npz --steps 5 > $A/bench_$c.json 2> $A/bench_$c.err
done
for cell in "nc=65536,nv=10000000,R=inf,D=inf" "nc=16384,nv=10000000,R=1,D=inf" "nc=4096,nv=10000000,R=0.2,D=0.5"; do
  python bench.py --workload raw --raw $cell --no-cpu-baseline --steps 5 > "$A/bench_raw_$cell.json" 2> "$A/bench_raw_$cell.err"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_cfg2.csv \
    python bench.py --greedy-cache devcache/cfg2_controls.npz --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_volume_exact_tiled --launch-skip 8 -c 1 \
    -o /tmp/k_exact python bench.py --greedy-cache devcache/cfg2_controls.npz --steps 2 --warmup 3 --no-cpu-baseline --no-fast > /dev/null 2>&1
ncu -i /tmp/k_exact.ncu-rep --page raw --csv > $A/ncu_exact_cfg2_raw.csv 2>/dev/null
ncu -i /tmp/k_exact.ncu-rep --page details --csv > $A/ncu_exact_cfg2_details.csv 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:k_volume_fast --launch-skip 2 -c 1 \
    -o /tmp/k_fast python bench.py --workload cfg4 --greedy-cache devcache/cfg4_controls.npz --precision fp64 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu -i /tmp/k_fast.ncu-rep --page raw --csv > $A/ncu_fast_cfg4_raw.csv 2>/dev/null
ncu -i /tmp/k_fast.ncu-rep --page details --csv > $A/ncu_fast_cfg4_details.csv 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:k_volume_f32 --launch-skip 2 -c 1 \
    -o /tmp/k_f32 python bench.py --workload raw --raw nc=65536,nv=10000000,R=inf,D=inf --precision fp32 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu -i /tmp/k_f32.ncu-rep --page raw --csv > $A/ncu_f32_raw_raw.csv 2>/dev/null
ncu -i /tmp/k_f32.ncu-rep --page details --csv > $A/ncu_f32_raw_details.csv 2>/dev/null
ls -la $A
