# usage (on a gpurun box with N GPUs): bash tools/mgpu_check.sh N
N=$1
python -m pytest tests/test_multigpu_gpu.py -q -x > gpurun_out/mp$N.log 2>&1; tail -3 gpurun_out/mp$N.log
for r in p2p nccl; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29612 bench.py --gpus $N --steps 20 --reduce $r --no-e2e \
    > gpurun_out/bench_n${N}_$r.log 2> gpurun_out/bench_n${N}_$r.err
  tail -c 1200 gpurun_out/bench_n${N}_$r.log
done
