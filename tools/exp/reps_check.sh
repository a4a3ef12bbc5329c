export PIER_ROUND_TIMEOUT_S=30
timeout 1200 python -m pytest tests/test_virtual_groups_gpu.py tests/test_multigpu_gpu.py -q -p no:cacheprovider -k "layout" > gpurun_out/reps_tests.log 2>&1; tail -3 gpurun_out/reps_tests.log; grep -E "^(FAILED|ERROR)|Error|assert" gpurun_out/reps_tests.log | head
LB_ARGS="--layouts 2x2x1" bash tools/exp/layout_bench.sh
