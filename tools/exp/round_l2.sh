# Result: n=2 B=4M 12.66 -> 12.45 ms with evict_last (kept, default); n=4 unchanged, B=2M 14.75 vs 4M 15.1 (bench auto bucket).
# AdamW-role theta stores: default write-back vs an L2 evict-last policy (PIER_ROUND_L2LAST)
run() { for N in 2 4; do for k in 1 2; do BUCKETS=2097152,4194304 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N tools/round_sweep.py --reps 10 2>/dev/null | grep "{"; done; done; }
echo "== default"; run
cd paper_2511_17849_b200/csrc && touch pier_round.cu && make EXTRA=-DPIER_ROUND_L2LAST > /dev/null 2>&1; cd ../..
echo "== evict_last"; run
