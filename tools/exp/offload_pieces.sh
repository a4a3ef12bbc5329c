# offload parks/fetches in 64 MB pieces on separate D2H / H2D streams (4-GPU box)
python -m pytest tests/test_kernels_gpu.py tests/test_configs_gpu.py tests/test_multigpu_gpu.py -q -x > gpurun_out/off_tests.log 2>&1; tail -2 gpurun_out/off_tests.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29702 tools/config_bench.py --config medium --compare-offload 2>/dev/null | grep "{"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29703 tools/config_bench.py --config 7b --compare-offload 2>/dev/null | grep "{"
