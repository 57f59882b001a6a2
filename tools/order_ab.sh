# spatial order A/B (diagnostic): Morton (default) vs grid cells, exact and fast
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
for o in morton grid; do for p in exact fp64; do for c in cfg2 cfg3; do
  IMB_ORDER=$o python bench.py --workload $c --greedy-cache devcache/${c}_controls.npz --no-cpu-baseline --no-fast --steps 3 --precision $p 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$o', d['config']['workload'], d['config']['precision'], d['value'], d['roofline']['frac'], d['kernel_ms_avg'], 'e2e', d['e2e']['value'])"
done; done; done
