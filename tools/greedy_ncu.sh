# ncu evidence for the exact greedy kernels: k_backward_t (chain, n = 4096),
# k_sweep and k_insert at a late step of cfg2 level 1, and the launch list of
# cfg2 levels 0-1 (per-kernel shares of a greedy level).
A=gpurun_out/greedy; mkdir -p $A
python tools/chain_ncu.py 4096 > $A/chain.log 2>&1; cat $A/chain.log
python tools/greedy_levels.py cfg2 2 > $A/levels.log 2>&1; cat $A/levels.log
ncu --set full --import-source on --clock-control none -k regex:k_backward_t --launch-skip 2 -c 1 -o /tmp/bw python tools/chain_ncu.py 4096 > $A/ncu_bw.log 2>&1
ncu -i /tmp/bw.ncu-rep --page raw --csv > $A/ncu_backward_raw.csv 2>/dev/null
ncu -i /tmp/bw.ncu-rep --page details --csv > $A/ncu_backward_details.csv 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:"k_sweep|k_insert" --launch-skip 2400 -c 2 -o /tmp/sw python tools/greedy_levels.py cfg2 2 > $A/ncu_sw.log 2>&1
ncu -i /tmp/sw.ncu-rep --page raw --csv > $A/ncu_sweep_insert_raw.csv 2>/dev/null
ncu -i /tmp/sw.ncu-rep --page details --csv > $A/ncu_sweep_insert_details.csv 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_greedy_cfg2.csv python tools/greedy_levels.py cfg2 2 > $A/ncu_ll.log 2>&1
ls -la $A
