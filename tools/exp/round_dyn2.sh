# Experiment record (see round_dyn.sh): the switches are gone; kept for the numbers in DESIGN.md.
run() { for N in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N tools/round_sweep.py --reps 10 2>/dev/null | grep "{"; done; }
cd paper_2511_17849_b200/csrc && touch pier_round.cu && make EXTRA=-DPIER_ROUND_MIN_CTAS=4 > /dev/null 2>&1; cd ../..
echo "== min4 dyn"; PIER_ROUND_DYN=1 BUCKETS=2097152,4194304,8388608 SPLITS=3:0 run
cd paper_2511_17849_b200/csrc && touch pier_round.cu && make EXTRA=-DPIER_ROUND_MIN_CTAS=5 > /dev/null 2>&1; grep -A1 "k_round" build/pier_round.ptxas.txt | grep -i spill | sort | uniq -c; cd ../..
echo "== min5 dyn"; PIER_ROUND_DYN=1 BUCKETS=4194304 SPLITS=4:0,3:296 run
