export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_cholesky.py -x -q > gpurun_out/pytest_chol.log 2>&1; echo rc=$? >> gpurun_out/pytest_chol.log
tail -n 25 gpurun_out/pytest_chol.log
SPEC_SEQ=0 timeout 900 python tools/spec_check.py cfg3l0 cfg4l01 > gpurun_out/spec_big.log 2>&1
cat gpurun_out/spec_big.log
