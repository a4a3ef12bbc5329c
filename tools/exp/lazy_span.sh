# span-layout sharded lazy steps + copy-engine overlap: tests (virtual + real ranks, raw ABI), lazy timing, overlap bench
export PIER_ROUND_TIMEOUT_S=30
timeout 1500 python -m pytest tests/test_virtual_groups_gpu.py tests/test_multigpu_gpu.py tests/test_capi_gpu.py -q -p no:cacheprovider > gpurun_out/span_tests.log 2>&1; tail -3 gpurun_out/span_tests.log; grep -E "^(FAILED|ERROR)|Error|assert" gpurun_out/span_tests.log | head
for N in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N tools/round_ranks.py --steps 6 --lazy-ctas 6 2>/dev/null | grep -o '{"rank": 0, "world": [0-9], "lazy[^}]*}}'; done
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N tools/lazy_overlap_bench.py --steps 4 2>gpurun_out/ovl_n$N.err | grep "{"; tail -2 gpurun_out/ovl_n$N.err | grep -v OMP
done
