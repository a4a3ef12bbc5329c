# experiment: idle exchange CTAs run AdamW tiles while they wait (PIER_ROUND_HELP=1) vs the split roles
export PIER_ROUND_TIMEOUT_S=30
PIER_ROUND_HELP=1 timeout 900 python -m pytest tests/test_multigpu_gpu.py -q -p no:cacheprovider > gpurun_out/help_tests.log 2>&1; tail -2 gpurun_out/help_tests.log; grep -E "^(FAILED|ERROR)|Error|assert" gpurun_out/help_tests.log | head -5
for rep in 1 2; do for N in 2 4; do for H in 0 1; do
PIER_ROUND_HELP=$H timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N tools/round_ranks.py --steps 20 > gpurun_out/h$H$N.out 2>&1
python - <<PY
import json
for l in open("gpurun_out/h$H$N.out"):
    for x in l.replace("}{", "}\n{").splitlines():
        if x.startswith('{"rank": 0'):
            d = json.loads(x); print("help=$H", d["world"], d["round_ms_stats"], d["replicas_agree"])
PY
done; done; done
