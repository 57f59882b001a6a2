# gathered vs group-culled exact kernel (diagnostic)
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
for g in "" "IMB_NO_GATHER=1"; do for c in cfg2 cfg3 cfg4; do
  env $g python bench.py --workload $c --greedy-cache devcache/${c}_controls.npz --no-cpu-baseline --no-fast --steps 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('${g:-gather}', d['config']['workload'], d['config']['precision'], d['value'], d['roofline']['frac'], d['kernel_ms_avg'], 'e2e', d['e2e']['value'])"
done; done
