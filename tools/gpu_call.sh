set -x
export PYTHONUNBUFFERED=1
timeout 600 python tools/spec_check.py cfg1 cfg2l01 cfg3p cfg4p > gpurun_out/spec_check.log 2>&1; echo rc=$? >> gpurun_out/spec_check.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/pytest_all.log
tail -n 5 gpurun_out/pytest_all.log
cat gpurun_out/spec_check.log | grep -v "^\[spec\]" | tail -n 20
