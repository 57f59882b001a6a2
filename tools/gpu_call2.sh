export PYTHONUNBUFFERED=1
SPEC_SEQ=0 timeout 900 python tools/spec_check.py cfg4l01 cfg3l0 > gpurun_out/spec_big.log 2>&1
cat gpurun_out/spec_big.log
