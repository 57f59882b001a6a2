# FP64 fast path: Newton-only sqrt refinement (IMB_K1_EXP=N1, 15 FP64
# instructions per pair) vs the second-order correction (16), dense raw cell;
# parity of N1 against the 1e-10 bar on the raw / interpolant tests.
mkdir -p gpurun_out/n1
cell="nc=65536,nv=10000000,R=inf,D=inf"
for v in base N1 base N1; do
  IMB_K1_EXP=$v timeout 300 python bench.py --workload raw --raw $cell --precision fp64 \
    --no-cpu-baseline --steps 5 > gpurun_out/n1/$v.json 2> gpurun_out/n1/$v.err
  python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], d['value'], d['roofline']['frac'], d['kernel_ms_avg'])" gpurun_out/n1/$v.json $v || tail -3 gpurun_out/n1/$v.err
done
IMB_K1_EXP=N1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "raw or interpolant or deform" > gpurun_out/n1/pytest_n1.log 2>&1
tail -3 gpurun_out/n1/pytest_n1.log
