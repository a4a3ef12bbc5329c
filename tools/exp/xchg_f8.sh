# Result (4 GPUs, XL, B=4M): float4 14.95-14.97 ms, F8 15.83-15.87 ms -> kept float4 (macro removed).
# exchange-role vector width at n = 3..4: float4 (default) vs F8 (PIER_XCHG_F8_MAX=4)
run() { for N in 4; do for k in 1 2; do BUCKETS=4194304 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N tools/round_sweep.py --reps 10 2>/dev/null | grep "{"; done; done; }
echo "== float4"; run
cd paper_2511_17849_b200/csrc && touch pier_round.cu && make EXTRA=-DPIER_XCHG_F8_MAX=4 > /dev/null 2>&1; cd ../..
echo "== F8"; run
