# Exact tiled kernel: occupancy / controls-per-stage variants (IMB_XT_EXP)
# vs the default (6 CTAs/SM, 2 controls x 2 points), exact precision.
A=gpurun_out/xt; mkdir -p $A
for rep in 1 2; do
for v in base m5 m4 m4c4; do
  for w in cfg2 cfg3 cfg4; do
    IMB_XT_EXP=$v timeout 600 python bench.py --workload $w --greedy-cache devcache/${w}_controls.npz --no-fast --no-cpu-baseline --steps 3 > $A/${w}_$v.$rep.json 2>$A/${w}_$v.$rep.err
    python -c "import json,sys; d=json.load(open('$A/${w}_$v.$rep.json')); print('$w', '$v', $rep, round(d['value'],1), d['roofline']['frac'], d['kernel_ms_avg'])" || echo "$w $v fail"
  done
done
done
