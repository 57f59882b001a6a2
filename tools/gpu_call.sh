export PYTHONUNBUFFERED=1 IMB_SPEC_WATCHDOG_S=20
timeout 300 python tools/spec_check.py cfg1 cfg2l01 cfg3p cfg4p > gpurun_out/a.log 2>&1
grep -v "^\[spec\]  k=" gpurun_out/a.log | tail -n 30
