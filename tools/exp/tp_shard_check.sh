# sharded steps with tensor parallelism: the layout tests (virtual 4/8 ranks + real 4 ranks), then the layout bench
timeout 1200 python -m pytest tests/test_virtual_groups_gpu.py tests/test_multigpu_gpu.py -q -p no:cacheprovider -k "layout" > gpurun_out/tp_tests.log 2>&1; tail -3 gpurun_out/tp_tests.log; grep -E "^(FAILED|ERROR)|Error|assert" gpurun_out/tp_tests.log | head
bash tools/exp/layout_bench.sh
