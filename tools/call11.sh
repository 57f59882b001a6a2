# k_insert with a 4-column cp.async ring: parity (all GPU tests, the 2-column
# fallback on the greedy tests, the full cfg2 selection) and timing
A=gpurun_out/c11; mkdir -p $A
timeout 900 python -m pytest tests -m gpu -q -x > $A/pytest.log 2>&1; tail -1 $A/pytest.log
IMB_INSERT_RING2=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $A/pytest_ring2.log 2>&1; tail -1 $A/pytest_ring2.log
python tools/greedy_levels.py cfg2 2 > $A/staged.log 2>&1; cat $A/staged.log
IMB_FULL=1 timeout 1200 python -m pytest tests -m gpu -q -x -k "cfg2_full_selection" > $A/pytest_full.log 2>&1; tail -1 $A/pytest_full.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_greedy_cfg2.csv python tools/greedy_levels.py cfg2 2 > /dev/null 2>&1
