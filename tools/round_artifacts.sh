# Round-end measurement set (run on the GPU box through gpurun; everything
# lands in gpurun_out/art and is copied to profiles/ by hand).  gpurun_in/
# may hold exact greedy selections of an earlier device run (bench.py
# --greedy-cache) for the secondary lines; the default line runs the greedy
# on the device itself.
#   pytest -m gpu, smoke, default bench (cfg4, full), reference arm, cfg2 /
#   cfg3 lines, raw-sweep cells, ncu launch list of a cfg4 bench run, one
#   ncu --set full capture of the headline kernel and of the compaction
#   kernels (reports stay in /tmp, only CSV pages come back).
export PYTHONUNBUFFERED=1
A=gpurun_out/art
mkdir -p $A devcache
cp gpurun_in/*.npz devcache/ 2>/dev/null
python -m pytest tests -m gpu -q > $A/pytest_gpu.log 2>&1; tail -1 $A/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $A/smoke.log 2>&1; tail -1 $A/smoke.log
( time python bench.py > $A/bench_cfg4.json 2> $A/bench_cfg4.err ) 2> $A/bench_cfg4.time; tail -3 $A/bench_cfg4.time
( time python bench.py --impl reference > $A/bench_reference.json 2> $A/bench_reference.err ) 2> $A/bench_reference.time
for c in cfg2 cfg3; do
  python bench.py --workload $c --greedy-cache devcache/${c}_controls.npz --steps 5 > $A/bench_$c.json 2> $A/bench_$c.err
done
for cell in "nc=65536,nv=10000000,R=inf,D=inf" "nc=16384,nv=10000000,R=1,D=inf" "nc=4096,nv=10000000,R=0.2,D=0.5"; do
  python bench.py --workload raw --raw $cell --no-cpu-baseline --steps 5 > "$A/bench_raw_$cell.json" 2> "$A/bench_raw_$cell.err"
done
B="python bench.py --greedy-cache devcache/cfg4_controls.npz --steps 2 --warmup 1 --no-deform --no-cpu-baseline --no-fast"
$B > $A/plain_cfg4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $A/launches_cfg4.csv $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_volume_exact_tiled --launch-skip 1 -c 1 -o /tmp/k_exact -f $B > $A/ncu_exact.log 2>&1
ncu -i /tmp/k_exact.ncu-rep --page raw --csv > $A/ncu_k_volume_exact_tiled_cfg4_raw.csv 2>/dev/null
ncu -i /tmp/k_exact.ncu-rep --page details --csv > $A/ncu_k_volume_exact_tiled_cfg4_details.csv 2>/dev/null
python tools/hbm_passes.py cfg3 1.0 1.0 1 > $A/hbm_cfg3.json 2>&1 && \
ncu --set full --clock-control none -k regex:"k_compact_active" -c 3 -o /tmp/cp -f python tools/hbm_passes.py cfg3 1.0 1.0 1 > $A/ncu_cp.log 2>&1
ncu -i /tmp/cp.ncu-rep --page raw --csv > $A/ncu_k_compact_active_cfg3_raw.csv 2>/dev/null
ncu -i /tmp/cp.ncu-rep --page details --csv > $A/ncu_k_compact_active_cfg3_details.csv 2>/dev/null
du -sh gpurun_out; ls -la $A
