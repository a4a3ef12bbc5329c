# Experiment record: the static/dynamic AdamW-role switch (PIER_ROUND_DYN) and PIER_ROUND_MIN_CTAS
# were folded into the kernel (dynamic claiming, 4 CTAs/SM) after this measurement.
run() { for N in 2 4; do BUCKETS=4194304 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N tools/round_sweep.py --reps 10 2>/dev/null | grep "{"; done; }
echo "== min3 static"; SPLITS=2:0 run
echo "== min3 dyn"; PIER_ROUND_DYN=1 SPLITS=2:0 run
cd paper_2511_17849_b200/csrc && touch pier_round.cu && make EXTRA=-DPIER_ROUND_MIN_CTAS=4 > /dev/null 2>&1; grep -A1 "k_roundILi2" build/pier_round.ptxas.txt | tail -1; cd ../..
echo "== min4 static"; SPLITS=3:0,2:296 run
echo "== min4 dyn"; PIER_ROUND_DYN=1 SPLITS=3:0,2:296 run
