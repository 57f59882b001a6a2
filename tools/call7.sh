timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_c7.log 2>&1; tail -1 gpurun_out/pytest_c7.log
bash tools/greedy_ncu.sh
bash tools/round_artifacts.sh
