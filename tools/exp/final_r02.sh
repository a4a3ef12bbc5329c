# end-of-change evidence (4-GPU box): smoke, the whole GPU suite, bench n = 1 / 2 / 4 (self-launched)
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu4_tests.log 2>&1; tail -2 gpurun_out/gpu4_tests.log; grep -E "^(FAILED|ERROR)" gpurun_out/gpu4_tests.log | head
for N in 1 2 4; do timeout 900 python bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_n$N.json').read().strip().splitlines()[-1]); print(d['n_gpus'], d['ms_per_step'], d['roofline']['bound'], round(d['roofline']['frac'],3), d['clocks'], (d.get('lazy_phase') or {}).get('iteration_ms'), d['e2e']['ms_per_step'])"; done
