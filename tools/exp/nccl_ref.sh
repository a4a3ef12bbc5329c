# NCCL reference points at n = 2 and 4 (4-GPU box): plain all-reduce / RS+AG bus bandwidth of
# the XL buffer, and bench.py with the bucketed NCCL and NVLS exchanges instead of the P2P round
for N in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2990$N tools/nccl_busbw.py 2>/dev/null | grep "{"
  for r in nccl nvls; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2991$N bench.py --gpus $N --steps 20 --reduce $r --no-e2e --no-cpu 2>/dev/null | grep "{" > gpurun_out/bench_n${N}_$r.json
    python -c "import json; d=json.load(open('gpurun_out/bench_n${N}_$r.json')); print('N=$N reduce=$r', round(d['ms_per_step'],3), d['kernels_ms'])"
  done
done
