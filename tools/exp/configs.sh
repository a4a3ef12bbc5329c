# configs 2, 3, 5 + the reference arm + multi-tensor tests (4-GPU box)
python -m pytest tests/test_kernels_gpu.py -q -p no:cacheprovider -k "multi_tensor or mt" 2>&1 | tail -2
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29701 tools/config_bench.py --config small 2>/dev/null | grep "{"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29702 tools/config_bench.py --config medium --compare-offload 2>/dev/null | grep "{"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29703 tools/config_bench.py --config 7b --compare-offload 2>/dev/null | grep "{"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | tail -1
