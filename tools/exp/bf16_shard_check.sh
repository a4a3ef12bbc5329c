# bf16 (7B recipe) sharded lazy step: the multi-rank GPU tests, then 7B lazy / inner / boundary times at n = 2 / 4
export PIER_ROUND_TIMEOUT_S=30
timeout 1500 python -m pytest tests/test_virtual_groups_gpu.py tests/test_multigpu_gpu.py tests/test_capi_gpu.py tests/test_configs_gpu.py -q -p no:cacheprovider > gpurun_out/bf16_tests.log 2>&1; tail -3 gpurun_out/bf16_tests.log; grep -E "^(FAILED|ERROR)|Error|assert" gpurun_out/bf16_tests.log | head
bash tools/exp/bf16_lazy.sh
