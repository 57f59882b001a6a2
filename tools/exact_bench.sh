# GPU tests + exact-mode bench of cfg2/3/4 with the cached greedy selections (diagnostic)
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
for c in cfg2 cfg3 cfg4; do
  python bench.py --workload $c --greedy-cache devcache/${c}_controls.npz --no-cpu-baseline --steps 3 --precision ${PREC:-exact} 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['config']['workload'], d['config']['precision'], d['value'], d['roofline']['frac'], d['kernel_ms_avg'], 'e2e', d['e2e']['value'])"
done
