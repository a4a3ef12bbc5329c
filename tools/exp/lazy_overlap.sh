# the lazy step overlapped with a synthetic backward: correctness (virtual + real ranks), then timing at n = 2 / 4
timeout 1500 python -m pytest tests/test_virtual_groups_gpu.py tests/test_multigpu_gpu.py -q -p no:cacheprovider -k "engine_bitwise or outer" > gpurun_out/ovl_tests.log 2>&1; tail -3 gpurun_out/ovl_tests.log; grep -E "^(FAILED|ERROR)|Error|assert" gpurun_out/ovl_tests.log | head
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N tools/lazy_overlap_bench.py 2>gpurun_out/ovl_n$N.err | grep "{"; tail -2 gpurun_out/ovl_n$N.err
done
