# 7B recipe (bf16 params/grads, fp32 master/m/v): lazy / inner / boundary iteration times at n = 2 and 4 groups
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29712 tools/layout_bench.py --config 7b --bf16 --layouts 2x1x1 --steps 4 2>gpurun_out/bf16_n2.err | tee gpurun_out/bf16_lazy.jsonl
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29714 tools/layout_bench.py --config 7b --bf16 --layouts 4x1x1 --steps 4 2>gpurun_out/bf16_n4.err | tee -a gpurun_out/bf16_lazy.jsonl
tail -2 gpurun_out/bf16_n4.err
