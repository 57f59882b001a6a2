# A/B of the FP32 volume kernel variants (IMB_F32_EXP) on raw sweep cells.
mkdir -p gpurun_out/f32ab
for cell in "nc=65536,nv=10000000,R=inf,D=inf" "nc=16384,nv=10000000,R=1,D=inf"; do
  for v in base p2b2n4 p4b1n2 p2b3n2 p1b3n4 p2b2n1; do
    IMB_F32_EXP=$v timeout 300 python bench.py --workload raw --raw $cell --precision fp32 --no-fast \
      --no-cpu-baseline --steps 5 > gpurun_out/f32ab/$v.json 2> gpurun_out/f32ab/$v.err
    python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], sys.argv[3], d['value'], d['roofline']['frac'], d['kernel_ms_avg'])" gpurun_out/f32ab/$v.json "$cell" $v || tail -3 gpurun_out/f32ab/$v.err
  done
done
