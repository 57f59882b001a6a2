# k_insert CTA size A/B (IMB_INSERT_T): timing on cfg2 levels 0-1 + parity
A=gpurun_out/c14; mkdir -p $A
for t in 1024 512 256; do
  IMB_INSERT_T=$t python tools/greedy_levels.py cfg2 2 > $A/t$t.log 2>&1; echo "T=$t $(cat $A/t$t.log)"
done
for t in 512 256; do
  IMB_INSERT_T=$t timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $A/pytest_t$t.log 2>&1; echo "T=$t $(tail -1 $A/pytest_t$t.log)"
done
