# full -m gpu suite, smoke, then compute-sanitizer memcheck on the small cases
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_all.log 2>&1 ) 2> gpurun_out/pytest_all.time; echo rc=$? >> gpurun_out/pytest_all.log
tail -n 25 gpurun_out/pytest_all.log; cat gpurun_out/pytest_all.time
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 600 python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 7 python tools/sanitize_cases.py > gpurun_out/sanitize_memcheck.log 2>&1; echo memcheck rc=$?
tail -5 gpurun_out/sanitize_plain.log; tail -8 gpurun_out/sanitize_memcheck.log
