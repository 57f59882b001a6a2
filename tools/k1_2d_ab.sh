# FP64 fast kernel on planar (2-D) meshes: the default shape vs the 3-D
# lockstep shape (4 controls x 2 points, whole group per iteration), cfg2.
A=gpurun_out/ab2d; mkdir -p $A
for rep in 1 2; do
for v in default L2d2; do
  IMB_K1_EXP=$v timeout 600 python bench.py --workload cfg2 --greedy-cache devcache/cfg2_controls.npz --precision fp64 --no-cpu-baseline --steps 5 > $A/cfg2_$v.$rep.json 2>$A/cfg2_$v.$rep.err
  python -c "import json; d=json.load(open('$A/cfg2_$v.$rep.json')); print('cfg2', '$v', $rep, round(d['value'],1), d['roofline']['frac'], d['kernel_ms_avg'])" || echo "cfg2 $v fail"
done
done
IMB_K1_EXP=L2d2 timeout 900 python -m pytest tests -m gpu -q -x -k "fast or fp64 or interpolant or deform" > $A/pytest_l2d2.log 2>&1; tail -1 $A/pytest_l2d2.log
