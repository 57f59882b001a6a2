# A/B of K1 variants (diagnostic): grouped-ballot loop (default) vs unrolled groups
set -e
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "" "IMB_K1_UNROLLED_GROUPS=1"; do
  echo "variant: ${v:-loopg}"
  env $v python bench.py --workload raw --raw nc=4096,nv=10000000,R=inf,D=inf --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('raw3d', d['value'], d['roofline']['frac'], d['kernel_ms_avg'])"
  env $v python bench.py --workload raw --raw nc=16384,nv=10000000,R=1,D=0.5 --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('raw R1', d['value'], d['roofline']['frac'], d['kernel_ms_avg'])"
  env $v python bench.py --greedy-cache devcache/cfg2_controls.npz --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('cfg2', d['value'], d['roofline']['frac'], d['kernel_ms_avg'], d['e2e']['value'])"
done
