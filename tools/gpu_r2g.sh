export PYTHONUNBUFFERED=1
mkdir -p gpurun_out devcache
cp gpurun_in/*.npz devcache/ 2>/dev/null
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spec.py tests/test_gpu_wing.py tests/test_gpu_cholesky.py tests/test_gpu_pipeline.py -m gpu -x -q > gpurun_out/pytest_sweep.log 2>&1; echo rc=$? >> gpurun_out/pytest_sweep.log
tail -n 4 gpurun_out/pytest_sweep.log
timeout 600 python tools/greedy_levels.py cfg3 1 > gpurun_out/greedy_cfg3.log 2>&1; tail -1 gpurun_out/greedy_cfg3.log
IMB_SPEC=0 timeout 600 python tools/greedy_levels.py cfg2 2 > gpurun_out/greedy_cfg2_seq.log 2>&1 && \
IMB_SPEC=0 ncu --set full --clock-control none --import-source on -k regex:"k_sweep" --launch-skip 1200 -c 1 -o /tmp/sw -f python tools/greedy_levels.py cfg2 2 > gpurun_out/ncu_sw.log 2>&1
ncu -i /tmp/sw.ncu-rep --page raw --csv > gpurun_out/ncu_k_sweep_cfg2_raw.csv 2>/dev/null
ncu -i /tmp/sw.ncu-rep --page details --csv > gpurun_out/ncu_k_sweep_cfg2_details.csv 2>/dev/null
# the same kernel on the cfg3 surface (40k points), k ~ 1000: sequential engine, capped at 1100 points
IMB_SPEC=0 timeout 900 python tools/greedy_levels.py cfg3 1 1100 > gpurun_out/greedy_cfg3_seq.log 2>&1 && \
IMB_SPEC=0 ncu --set full --clock-control none -k regex:"k_sweep" --launch-skip 1000 -c 1 -o /tmp/sw3 -f python tools/greedy_levels.py cfg3 1 1100 > gpurun_out/ncu_sw3.log 2>&1
ncu -i /tmp/sw3.ncu-rep --page raw --csv > gpurun_out/ncu_k_sweep_cfg3_raw.csv 2>/dev/null
ncu -i /tmp/sw3.ncu-rep --page details --csv > gpurun_out/ncu_k_sweep_cfg3_details.csv 2>/dev/null
tail -2 gpurun_out/greedy_cfg3_seq.log
du -sh gpurun_out
