set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu4_tests.log 2>&1; tail -3 gpurun_out/gpu4_tests.log
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -c 3000 gpurun_out/bench_n1.json
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2981$N bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; tail -c 3000 gpurun_out/bench_n$N.json
done
