# A/B of the tile ring: warp release (default) vs one __syncthreads per tile
# (IMB_TILE_SYNC=1), on the volume kernels of cfg2 (exact + fast), cfg3
# (exact, gathered kernel), cfg4 (exact + fast) and the dense raw cell (FP32).
mkdir -p gpurun_out/syncab
run() {  # name, env, bench args...
  local name=$1 envv=$2; shift 2
  env $envv timeout 900 python bench.py "$@" --no-cpu-baseline > gpurun_out/syncab/$name.json 2> gpurun_out/syncab/$name.err
  python -c "import json,sys; d=json.load(open(sys.argv[1])); f=d.get('fp64_fast') or {}; g=d.get('fp32') or {}; print(sys.argv[2], d['value'], d['kernel_ms_avg'], f.get('value'), f.get('kernel_ms_avg'), g.get('value'))" gpurun_out/syncab/$name.json $name || tail -3 gpurun_out/syncab/$name.err
}
for v in "A IMB_TILE_SYNC=1" "B IMB_NONE=1" "A2 IMB_TILE_SYNC=1" "B2 IMB_NONE=1"; do
  set -- $v
  run cfg2_$1 $2 --greedy-cache devcache/cfg2_controls.npz --steps 10
  run cfg3_$1 $2 --workload cfg3 --greedy-cache devcache/cfg3_controls.npz --steps 5
  run cfg4_$1 $2 --workload cfg4 --greedy-cache devcache/cfg4_controls.npz --steps 2
  run raw_$1 $2 --workload raw --raw nc=65536,nv=10000000,R=inf,D=inf --steps 3
done
