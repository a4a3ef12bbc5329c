# end-of-session evidence run (4-GPU box): smoke, full GPU suite, bench n=1/2/4; CONFIGS=1 adds configs 2/3/5
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
bash tools/gpu_round_check.sh 2>/dev/null
if [ "${CONFIGS:-0}" = "1" ]; then bash tools/exp/configs.sh > gpurun_out/configs_final.log 2>&1; cut -c1-300 gpurun_out/configs_final.log; fi
