A=gpurun_out/c15; mkdir -p $A
for t in 256 1024 512; do
  IMB_INSERT_T=$t python tools/greedy_levels.py cfg2 3 > $A/t$t.log 2>&1; echo "T=$t $(cat $A/t$t.log)"
done
