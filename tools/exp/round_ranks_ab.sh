for rep in 1 2; do for N in 4 2; do for F in "" "--no-lazy-shard"; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N tools/round_ranks.py $F 2>/dev/null | grep '"rank": 0'
done; done; done
