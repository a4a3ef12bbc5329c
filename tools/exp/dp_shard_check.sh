# dp-team sharded inner steps: the layout tests (virtual 4/8 ranks + real 4 ranks), the C-ABI tests, then the layout bench
timeout 1200 python -m pytest tests/test_virtual_groups_gpu.py tests/test_multigpu_gpu.py tests/test_capi_gpu.py -q -p no:cacheprovider -k "layout or topolog or capi or raw" > gpurun_out/dp_tests.log 2>&1; tail -3 gpurun_out/dp_tests.log; grep -E "^(FAILED|ERROR)|Error" gpurun_out/dp_tests.log | head
bash tools/exp/layout_bench.sh
