# exact 3-D: 4 controls per stage for whole groups only (default) vs for
# every batch (IMB_XT_EXP=c4) vs round-1 (base)
A=gpurun_out/c9; mkdir -p $A
timeout 900 python -m pytest tests -m gpu -q -x > $A/pytest.log 2>&1; tail -1 $A/pytest.log
for rep in 1 2; do
for v in default c4 base; do
  IMB_XT_EXP=$v timeout 600 python bench.py --workload cfg4 --greedy-cache devcache/cfg4_controls.npz --no-fast --no-cpu-baseline --steps 3 > $A/cfg4_$v.$rep.json 2>$A/cfg4_$v.$rep.err
  python -c "import json; d=json.load(open('$A/cfg4_$v.$rep.json')); print('cfg4', '$v', $rep, round(d['value'],1), d['roofline']['frac'], d['kernel_ms_avg'])" || echo "cfg4 $v fail"
  for cell in "nc=16384,nv=10000000,R=1,D=inf" "nc=4096,nv=10000000,R=0.2,D=0.5"; do
    IMB_XT_EXP=$v timeout 600 python bench.py --workload raw --raw $cell --no-fast --no-cpu-baseline --steps 3 > "$A/raw_$cell.$v.$rep.json" 2>/dev/null
    python -c "import json; d=json.load(open('$A/raw_$cell.$v.$rep.json')); print('$cell', '$v', $rep, round(d['value'],1), d['roofline']['frac'], d['kernel_ms_avg'])" || echo "raw $v fail"
  done
done
done
