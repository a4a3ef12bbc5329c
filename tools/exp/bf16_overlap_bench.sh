for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N tools/lazy_overlap_bench.py --steps 4 --bf16 2>gpurun_out/bovl_n$N.err | grep "{"; tail -3 gpurun_out/bovl_n$N.err | grep -v OMP
done
