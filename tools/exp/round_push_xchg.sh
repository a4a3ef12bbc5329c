# RESULT (r01, 4 B200): an all-writes exchange role -- once the local AdamW passed
# span b, the exchange CTAs copy every peer's slice into that peer's staging buffer
# (NVLink writes) and bump its arrived[b]; they then fold span b-1 from local memory
# (own slice + staging) and push the results.  Bitwise-correct (tests/test_multigpu_gpu.py
# 7 passed with PIER_ROUND_PUSH=1), but SLOWER than the pull round on the same box:
#   n=4: round 15.80 vs 13.88 ms (step 16.72 vs 14.82); n=2: 12.70-12.76 vs 11.54-11.57 ms.
# The staging write + re-read adds 8(n-1)/n B/param of HBM traffic and each exchange
# CTA alternates send and fold instead of streaming one pattern; the 4 % higher
# write-only link ceiling (profiles/r01_nvl_mix_probe_n4.jsonl) does not pay for it.
# Switch removed from the kernel after the measurement (commit message has the diff summary).
set -x
PIER_ROUND_PUSH=1 timeout 900 python -m pytest tests/test_multigpu_gpu.py -x -q > gpurun_out/push_mp.log 2>&1; tail -3 gpurun_out/push_mp.log
for N in 4 2; do
for P in 0 1 0 1; do
PIER_ROUND_PUSH=$P timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2975$N bench.py --gpus $N --steps 20 --no-e2e --no-cpu > gpurun_out/push_b${N}_${P}.json 2>gpurun_out/push_b.err
python -c "import json,sys; d=json.loads([l for l in open('gpurun_out/push_b${N}_${P}.json') if l.startswith('{')][-1]); print('N=$N push=$P', round(d['ms_per_step'],3), d['kernels_ms']['timed_step'], d['roofline']['bound'], round(d['roofline']['frac'],3))"
done
done
