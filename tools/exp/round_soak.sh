# soak: 300 consecutive XL Pier rounds (K4a + persistent round) on 2 and 4 real ranks; per-round distribution
for N in 4 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N tools/round_ranks.py --steps 300 > gpurun_out/soak_n$N.out 2>gpurun_out/soak_n$N.err
python - <<PY
import json
for l in open("gpurun_out/soak_n$N.out"):
    for x in l.replace("}{", "}\n{").splitlines():
        if x.startswith("{"):
            d = json.loads(x)
            print(json.dumps({k: d[k] for k in ("rank", "world", "round_ms_stats", "replicas_agree", "params_checksum")}))
PY
done
