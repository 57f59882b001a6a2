A=gpurun_out/c18; mkdir -p $A
python bench.py > $A/bench_cfg2.json 2> $A/bench_cfg2.err; echo rc=$?; tail -3 $A/bench_cfg2.err
python -c "import json; d=json.load(open('$A/bench_cfg2.json')); print(d['value'], d['e2e']['value'], d['greedy_seconds_per_level'], d['deform'])"
