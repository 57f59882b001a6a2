# cfg4 (3-D global, all in support) with the cached greedy selection: K1 variants
for v in L0 L2; do
  echo "exp=$v"
  IMB_K1_EXP=$v python bench.py --workload cfg4 --greedy-cache devcache/cfg4_controls.npz --no-cpu-baseline --steps 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('cfg4', d['value'], d['roofline']['frac'], d['kernel_ms_avg'], 'e2e', d['e2e']['value'])"
done
