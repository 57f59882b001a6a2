# final verification of the round's code: GPU suite, smoke, ncu of the FP32 kernel
A=gpurun_out/c17; mkdir -p $A
timeout 900 python -m pytest tests -m gpu -q > $A/pytest_gpu.log 2>&1; tail -1 $A/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $A/smoke.log 2>&1; tail -1 $A/smoke.log
ncu --set full --import-source on --clock-control none -k regex:k_volume_f32 --launch-skip 2 -c 1 \
    -o /tmp/k_f32 python bench.py --workload raw --raw nc=65536,nv=10000000,R=inf,D=inf --precision fp32 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu -i /tmp/k_f32.ncu-rep --page raw --csv > $A/ncu_f32_raw_raw.csv 2>/dev/null
ncu -i /tmp/k_f32.ncu-rep --page details --csv > $A/ncu_f32_raw_details.csv 2>/dev/null
python bench.py --workload raw --raw nc=65536,nv=10000000,R=inf,D=inf --precision fp32 --no-cpu-baseline --steps 5 > $A/bench_raw_fp32.json 2>/dev/null; cat $A/bench_raw_fp32.json | head -c 400
