export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 1500 python bench.py --greedy-cache gpurun_out/cfg4_sel.npz > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err ) 2> gpurun_out/bench_cfg4.time
tail -c 3000 gpurun_out/bench_cfg4.json; cat gpurun_out/bench_cfg4.time; tail -5 gpurun_out/bench_cfg4.err
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --steps 2 --warmup 1 --greedy-cache gpurun_out/cfg4_sel.npz --no-deform --no-cpu-baseline --no-fast > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
$NCU --set full --clock-control none --import-source on -k regex:k_volume_exact --launch-skip 1 -c 1 -o gpurun_out/ncu_exact_cfg4 -f python bench.py --steps 1 --warmup 1 --greedy-cache gpurun_out/cfg4_sel.npz --no-deform --no-cpu-baseline --no-fast > gpurun_out/ncu_exact.log 2>&1; echo exact rc=$?
$NCU --set full --clock-control none --import-source on -k regex:"k_wall_distance|k_count_active|k_scatter_active|k_scan_counts" -c 8 -o gpurun_out/ncu_hbm_cfg4 -f python bench.py --steps 1 --warmup 1 --greedy-cache gpurun_out/cfg4_sel.npz --no-deform --no-cpu-baseline --no-fast > gpurun_out/ncu_hbm.log 2>&1; echo hbm rc=$?
ls -la gpurun_out/*.ncu-rep
