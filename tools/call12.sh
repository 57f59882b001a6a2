bash tools/call11.sh
bash tools/greedy_ncu.sh
bash tools/round_artifacts.sh
