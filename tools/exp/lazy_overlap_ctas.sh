for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N tools/lazy_overlap_bench.py --ctas 1,2,6 --steps 4 2>gpurun_out/ovl_n$N.err | grep "{"; tail -2 gpurun_out/ovl_n$N.err | grep -v OMP
done
