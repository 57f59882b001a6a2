# FP32 kernel: clamp-free fully-inner groups (default) vs clamp everywhere
A=gpurun_out/c16; mkdir -p $A
timeout 900 python -m pytest tests/test_gpu_fp32.py -m gpu -q -x > $A/pytest.log 2>&1; tail -1 $A/pytest.log
for rep in 1 2; do
for v in default clampall; do
  for cell in "nc=65536,nv=10000000,R=inf,D=inf" "nc=16384,nv=10000000,R=1,D=inf"; do
    if [ $v = clampall ]; then export IMB_F32_CLAMP_ALL=1; else unset IMB_F32_CLAMP_ALL; fi
    timeout 600 python bench.py --workload raw --raw $cell --precision fp32 --no-cpu-baseline --steps 3 > "$A/$cell.$v.$rep.json" 2>/dev/null
    python -c "import json; d=json.load(open('$A/$cell.$v.$rep.json')); print('$cell', '$v', $rep, round(d['value'],1), d['roofline']['frac'], d['kernel_ms_avg'])" || echo "$cell $v fail"
  done
done
done
