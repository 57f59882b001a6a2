export PYTHONUNBUFFERED=1
A=gpurun_out/art5; mkdir -p $A devcache; cp gpurun_in/*.npz devcache/ 2>/dev/null
for f in 0.15 10; do
  IMB_GATHER_FRAC=$f python bench.py --workload cfg2 --greedy-cache devcache/cfg2_controls.npz --steps 5 --no-deform --no-cpu-baseline --no-fast > $A/bench_cfg2_f$f.json 2> $A/bench_cfg2_f$f.err
  IMB_GATHER_FRAC=$f python bench.py --workload raw --raw nc=16384,nv=10000000,R=1,D=inf --no-cpu-baseline --no-fast --steps 5 > $A/bench_rawR1_f$f.json 2> $A/bench_rawR1_f$f.err
  IMB_GATHER_FRAC=$f python bench.py --workload raw --raw nc=4096,nv=10000000,R=0.2,D=0.5 --no-cpu-baseline --no-fast --steps 5 > $A/bench_rawR02_f$f.json 2> $A/bench_rawR02_f$f.err
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/art5/bench_*.json")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["value"], d["roofline"]["frac"], d.get("kernel_ms_avg"))
PY
B="python bench.py --workload cfg2 --greedy-cache devcache/cfg2_controls.npz --steps 2 --warmup 1 --no-deform --no-cpu-baseline --no-fast"
$B > $A/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $A/launches_cfg2.csv $B > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_volume_exact_tiled --launch-skip 5 -c 1 -o /tmp/k2 -f $B > $A/ncu_k2.log 2>&1
ncu -i /tmp/k2.ncu-rep --page raw --csv > $A/ncu_k_volume_exact_tiled_cfg2_raw.csv 2>/dev/null
ncu -i /tmp/k2.ncu-rep --page details --csv > $A/ncu_k_volume_exact_tiled_cfg2_details.csv 2>/dev/null
