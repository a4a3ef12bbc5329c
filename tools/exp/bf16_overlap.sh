export PIER_ROUND_TIMEOUT_S=30
timeout 1500 python -m pytest tests/test_virtual_groups_gpu.py tests/test_multigpu_gpu.py -q -p no:cacheprovider -k "engine_bitwise or outer" > gpurun_out/bf16ovl_tests.log 2>&1; tail -3 gpurun_out/bf16ovl_tests.log; grep -E "^(FAILED|ERROR)|Error|assert" gpurun_out/bf16ovl_tests.log | head
