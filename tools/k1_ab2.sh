# FP64 fast kernel (3-D C2) launch-shape A/B: points per thread x controls per
# stage x unroll, on cfg4 (all pairs in support) and the dense raw cell.
VARIANTS=${VARIANTS:-"base L2p4c2 p4c2u2 p2c4u2 N1"}
A=gpurun_out/ab2; mkdir -p $A
for rep in 1 2; do
for v in $VARIANTS; do
  e=$v; [ $v = base ] && e=L2; [ $v = new ] && e=none
  IMB_K1_EXP=$e timeout 600 python bench.py --workload cfg4 --greedy-cache devcache/cfg4_controls.npz --precision fp64 --no-cpu-baseline --steps 3 > $A/cfg4_$v.$rep.json 2>$A/cfg4_$v.$rep.err
  IMB_K1_EXP=$e timeout 600 python bench.py --workload raw --raw nc=16384,nv=10000000,R=inf,D=inf --precision fp64 --no-cpu-baseline --steps 3 > $A/raw_$v.$rep.json 2>$A/raw_$v.$rep.err
  python - $A $v $rep <<'PY'
import json,sys
A,v,r=sys.argv[1:]
for w in ('cfg4','raw'):
    try:
        d=json.load(open(f'{A}/{w}_{v}.{r}.json'))
        print(w, v, r, round(d['value'],1), d['roofline']['frac'], d.get('kernel_ms_avg'), d['clocks']['sm_mhz'])
    except Exception as ex: print(w, v, r, 'fail', ex)
PY
done
done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/ab2/pytest_gpu.log 2>&1; tail -1 gpurun_out/ab2/pytest_gpu.log
