# Experiment record: the push-only round variant (round_impl="push") it compared was removed after
# this measurement; rerunning it now compares persistent vs streams.
timeout 300 python -m pytest tests/test_round_virtual_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -2
for N in 2 4; do
for I in persistent push persistent push; do IMPL=$I BUCKETS=4194304 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N tools/round_sweep.py --reps 10 2>/dev/null | grep "{"; done; done
timeout 700 python -m pytest tests/test_multigpu_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
