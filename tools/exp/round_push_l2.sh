# Result: no difference (n=2 12.45 vs 12.46, n=4 14.88 vs 14.88) -> not kept (macro removed).
# exchange-role result pushes: st.cg vs st.cg with an L2 evict-first policy (PIER_PUSH_EVICT_FIRST)
run() { for N in 2 4; do for k in 1 2; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N tools/round_sweep.py --reps 10 2>/dev/null | grep "{"; done; done; }
echo "== default"; BUCKETS=4194304 run
cd paper_2511_17849_b200/csrc && touch pier_round.cu && make EXTRA=-DPIER_PUSH_EVICT_FIRST > /dev/null 2>&1; cd ../..
echo "== evict_first pushes"; BUCKETS=4194304 run
