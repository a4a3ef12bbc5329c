# RESULT (r01, 4 B200): bucketed NCCL RS -> K3 -> AG outer step (bench.py --reduce nccl), ms of the
# outer step (unfused breakdown), span slice size x K3 grid cap (CTAs/SM, 0 = uncapped; a temporary
# PIER_NCCL_K3_CAP switch in pier_comm.cu, removed after this sweep):
#   n=4: 64 MB 17.0-19.0 | 256 MB 16.4 (cap 2: 17.0, cap 1: 17.1);  16 MB (bench default then): 28.0
#   n=2: 64 MB 17.0 (cap 2: 18.3) | 256 MB 15.0 (cap 2: 15.8, cap 1: 16.0); 16 MB: 22.8
# Capping K3 to leave SMs to NCCL does not help; large buckets do -> bench.py uses 256 MB for nccl.
# Plain NCCL on the same buffer (tools/nccl_busbw.py): all-reduce 10.05 / 13.85 ms, RS+AG 12.2 / 14.9 ms
# at n = 2 / 4 -- the P2P persistent round does AdamW AND the outer step in 11.55 / 13.9 ms.
for N in 4 2; do
for cfg in "64 0" "64 2" "256 0" "256 2" "256 1"; do
  set -- $cfg
  PIER_NCCL_K3_CAP=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2992$N bench.py --gpus $N --steps 10 --breakdown-steps 3 --reduce nccl --bucket-mb $1 --no-e2e --no-cpu 2>/dev/null | grep "{" > gpurun_out/nccl_sweep.json
  python -c "import json; d=json.load(open('gpurun_out/nccl_sweep.json')); print('N=$N bucket_mb=$1 cap=$2', round(d['ms_per_step'],3), round(d['kernels_ms']['unfused_breakdown']['outer_step'],3))"
done
done
