# groups x dp x tp layouts on 4 real ranks, XL: lazy / inner / outer iteration times (tools/layout_bench.py)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29714 tools/layout_bench.py ${LB_ARGS:-} 2>gpurun_out/layout_bench.err | tee gpurun_out/layout_bench.jsonl
tail -3 gpurun_out/layout_bench.err
