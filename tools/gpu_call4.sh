export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/pytest_all.log
tail -n 4 gpurun_out/pytest_all.log
( time timeout 1500 python bench.py --greedy-cache /tmp/cfg4_sel.npz > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err ) 2> gpurun_out/bench_cfg4.time
cat gpurun_out/bench_cfg4.time; tail -3 gpurun_out/bench_cfg4.err
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --steps 2 --warmup 1 --greedy-cache /tmp/cfg4_sel.npz --no-deform --no-cpu-baseline --no-fast > /tmp/ncu_launch.log 2>&1; echo launches rc=$?
$NCU --set full --clock-control none --import-source on -k regex:k_volume_exact --launch-skip 1 -c 1 -o /tmp/ncu_exact_cfg4 -f python bench.py --steps 1 --warmup 1 --greedy-cache /tmp/cfg4_sel.npz --no-deform --no-cpu-baseline --no-fast > /tmp/ncu_exact.log 2>&1; echo exact rc=$?
$NCU -i /tmp/ncu_exact_cfg4.ncu-rep --page raw --csv > gpurun_out/ncu_exact_cfg4_raw.csv 2>/dev/null
$NCU -i /tmp/ncu_exact_cfg4.ncu-rep --page details --csv > gpurun_out/ncu_exact_cfg4_details.csv 2>/dev/null
$NCU --set full --clock-control none -k regex:"k_wall_distance|k_count_active|k_scatter_active" -c 6 -o /tmp/ncu_hbm_cfg4 -f python bench.py --steps 1 --warmup 1 --greedy-cache /tmp/cfg4_sel.npz --no-deform --no-cpu-baseline --no-fast > /tmp/ncu_hbm.log 2>&1; echo hbm rc=$?
$NCU -i /tmp/ncu_hbm_cfg4.ncu-rep --page raw --csv > gpurun_out/ncu_hbm_cfg4_raw.csv 2>/dev/null
$NCU -i /tmp/ncu_hbm_cfg4.ncu-rep --page details --csv > gpurun_out/ncu_hbm_cfg4_details.csv 2>/dev/null
ls -la gpurun_out/
