# copy-engine overlap with the deferred all-gather: the lazy tests (virtual + real), then the bench
export PIER_ROUND_TIMEOUT_S=30
timeout 1500 python -m pytest tests/test_virtual_groups_gpu.py tests/test_multigpu_gpu.py -q -p no:cacheprovider > gpurun_out/ag_tests.log 2>&1; tail -3 gpurun_out/ag_tests.log; grep -E "^(FAILED|ERROR)|Error|assert" gpurun_out/ag_tests.log | head
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N tools/lazy_overlap_bench.py --steps 4 2>gpurun_out/ovl_n$N.err | grep "{"; tail -3 gpurun_out/ovl_n$N.err | grep -v OMP
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 tools/lazy_overlap_bench.py --steps 4 --layout 2x2x1 --phase outer 2>gpurun_out/ovl_dp.err | grep "{"
