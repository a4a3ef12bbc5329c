# experiment: AdamW role with two F8 vectors per thread per tile (k_round_u2, 3 CTAs/SM: 2 AdamW + 1 exchange)
# vs the default (k_round, 4 CTAs/SM: 3 + 1) -- live XL rounds on real ranks
for N in 2 4; do for U in 1 2; do
PIER_ROUND_U=$U timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N tools/round_ranks.py --steps 20 > gpurun_out/u$U$N.out 2>&1
python - <<PY
import json
for l in open("gpurun_out/u$U$N.out"):
    for x in l.replace("}{", "}\n{").splitlines():
        if x.startswith('{"rank": 0'):
            d = json.loads(x); print("U=$U", d["world"], d["round_ms_stats"], d["replicas_agree"])
PY
done; done
