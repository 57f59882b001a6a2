export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/pytest_all.log
tail -n 4 gpurun_out/pytest_all.log
./paper_2107_13887_b200/build/test_shim | tail -3
SPEC_SEQ=0 timeout 900 python tools/spec_check.py cfg3l0 cfg4l01 cfg2 > gpurun_out/spec_big.log 2>&1
cat gpurun_out/spec_big.log
