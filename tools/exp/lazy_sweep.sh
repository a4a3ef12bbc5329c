# sharded lazy step at n = 2 / 4 (XL): CTAs per SM of its exchange kernels (default 4), sharded vs replicated
for N in 2 4; do for F in "" "--no-lazy-shard"; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N tools/round_ranks.py --steps 6 --lazy-ctas 1,2,3,4,6,8 $F 2>/dev/null | grep -o '{"rank": 0, "world": [0-9], "lazy[^}]*}}'
done; done
