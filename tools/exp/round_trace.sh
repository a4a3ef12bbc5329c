cd paper_2511_17849_b200/csrc && touch pier_round.cu && make EXTRA=-DPIER_ROUND_TRACE > /dev/null 2>&1; cd ../..
for N in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N tools/exp/round_trace.py 2>/dev/null | grep "{"; done
