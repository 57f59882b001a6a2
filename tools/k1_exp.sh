# K1 3-D variants (diagnostic): IMB_K1_EXP selects the launch shape
#python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in L2 L2p4c2; do
  echo "exp=$v"
  IMB_K1_EXP=$v python bench.py --workload raw --raw nc=4096,nv=10000000,R=inf,D=inf --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('raw3d', d['value'], d['roofline']['frac'], d['kernel_ms_avg'])"
  IMB_K1_EXP=$v python bench.py --workload raw --raw nc=4096,nv=10000000,R=1,D=inf --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('raw3d R1', d['value'], d['roofline']['frac'], d['kernel_ms_avg'])"
done
