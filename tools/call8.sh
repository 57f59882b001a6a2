# register-budget A/B: 2-D fast kernel (IMB_K1_EXP=f2m2) on cfg2, gathered
# exact kernel (IMB_XG_EXP=m2) on cfg3
A=gpurun_out/c8; mkdir -p $A
for rep in 1 2; do
for v in default f2m2; do
  IMB_K1_EXP=$v timeout 600 python bench.py --workload cfg2 --greedy-cache devcache/cfg2_controls.npz --precision fp64 --no-cpu-baseline --steps 5 > $A/cfg2_$v.$rep.json 2>$A/cfg2_$v.$rep.err
  python -c "import json; d=json.load(open('$A/cfg2_$v.$rep.json')); print('cfg2 fp64', '$v', $rep, round(d['value'],1), d['roofline']['frac'], d['kernel_ms_avg'])" || echo "cfg2 $v fail"
done
for v in default m2; do
  IMB_XG_EXP=$v timeout 600 python bench.py --workload cfg3 --greedy-cache devcache/cfg3_controls.npz --no-fast --no-cpu-baseline --steps 5 > $A/cfg3_$v.$rep.json 2>$A/cfg3_$v.$rep.err
  python -c "import json; d=json.load(open('$A/cfg3_$v.$rep.json')); print('cfg3 exact', '$v', $rep, round(d['value'],1), d['roofline']['frac'], d['kernel_ms_avg'])" || echo "cfg3 $v fail"
done
done
