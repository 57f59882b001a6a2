# tiled exact kernel launch shapes (diagnostic): IMB_XT=<pts><ncl><minb>
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in 222 242 142 213 123 223 133; do
  echo "xt=$v"
  IMB_XT=$v python bench.py --workload cfg4 --greedy-cache devcache/cfg4_controls.npz --no-cpu-baseline --steps 2 --precision exact 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['config']['workload'], d['value'], d['roofline']['frac'], d['kernel_ms_avg'])"
done
