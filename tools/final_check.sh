python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
bash tools/gpu_round_check.sh 2>/dev/null
bash tools/exp/configs.sh > gpurun_out/configs_final.log 2>&1; cat gpurun_out/configs_final.log | cut -c1-300
