# 4-GPU box: the whole GPU suite (virtual groups + real 2/3/4-rank runs), then bench.py --gpus 2 / 4
nvidia-smi --query-gpu=name --format=csv,noheader | head -1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu4_tests.log 2>&1; tail -4 gpurun_out/gpu4_tests.log
grep -E "^(FAILED|ERROR)|Error" gpurun_out/gpu4_tests.log | head -20
for N in ${BENCH_NS:-2 4}; do timeout 600 python bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; tail -c 600 gpurun_out/bench_n$N.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_n$N.json').read().strip().splitlines()[-1]); print(d['n_gpus'], d['ms_per_step'], json.dumps(d.get('lazy_phase'))[:700])"; done
