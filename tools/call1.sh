A=gpurun_out/c1; mkdir -p $A gpurun_out/devcache
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $A/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x > $A/pytest_gpu.log 2>&1; tail -1 $A/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $A/smoke.log 2>&1; tail -1 $A/smoke.log
timeout 900 python bench.py --greedy-cache gpurun_out/devcache/cfg2_controls.npz > $A/bench_cfg2.json 2> $A/bench_cfg2.err; cat $A/bench_cfg2.json
for c in cfg3 cfg4; do
timeout 1200 python bench.py --workload $c --greedy-cache gpurun_out/devcache/${c}_controls.npz --steps 5 > $A/bench_$c.json 2> $A/bench_$c.err; cat $A/bench_$c.json
done
