# 7B recipe: fused bf16-gradient persistent round vs the unfused boundary (4-GPU box)
python -m pytest tests/test_multigpu_gpu.py -q -x > gpurun_out/bf16_mp.log 2>&1; tail -2 gpurun_out/bf16_mp.log
for u in "" "--unfused" "" "--unfused"; do
  echo "7b n=4 $u"
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29703 tools/config_bench.py --config 7b $u 2>/dev/null | grep "{" | cut -c1-400
done
