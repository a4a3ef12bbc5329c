for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2981$N bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; tail -1 gpurun_out/bench_n$N.json
done
bash tools/ncu_round.sh r01v8b > /dev/null 2>&1; ls gpurun_out | grep r01v8b
