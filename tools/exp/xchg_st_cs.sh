# RESULT (r01, 4 B200): no effect -- round (fused) ms, alternating .cg / .cs:
#   n=4: 13.81 / 13.80 / 13.81 (cg) vs 13.80 / 13.81 (cs);  n=2: 11.546 / 11.538 (cg) vs 11.566 / 11.562 (cs)
# The temporary PIER_XCHG_ST_CS switch was removed from pier_round.cu after the measurement.
# exchange result stores: .cg (current) vs .cs evict-first (PIER_XCHG_ST_CS=1), n = 4 and 2 (4-GPU box)
for N in 4 2; do
  if [ $N = 2 ]; then export CUDA_VISIBLE_DEVICES=0,1; fi
  for X in 0 1 0 1; do
    PIER_XCHG_ST_CS=$X timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2993$N bench.py --gpus $N --steps 30 --breakdown-steps 1 --no-e2e --no-cpu 2>/dev/null | grep "{" > gpurun_out/xcs.json
    python -c "import json; d=json.load(open('gpurun_out/xcs.json')); print('N=$N cs=$X', round(d['ms_per_step'],3), round(d['kernels_ms']['timed_step']['adamw+outer fused'],3))"
  done
done
