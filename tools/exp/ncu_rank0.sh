# RESULT (r01, 2 GPUs): did not work -- rank 0 under ncu never completed a profiled
# k_round within 420 s ("No kernels were profiled"); killed by timeout, no GPU fault.
# The round kernel's traffic stays null in bench.py.
# DRAM traffic of the multi-rank persistent round kernel (k_round): rank 0 runs
# bench.py under a SINGLE-PASS ncu collection (time + DRAM bytes need no kernel
# replay, so the cross-rank waits inside k_round see the same peers as an
# unprofiled run), every other rank runs bench.py plainly.
#   python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
#       --master-port 29733 --no-python bash tools/exp/ncu_rank0.sh N TAG
# A replayed (multi-pass) collection would deadlock the round's done-counter
# wait on rank 0; the kernel's 20 s spin guard then traps instead of hanging.
N=$1
TAG=${2:-r01}
ARGS="bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-cpu --breakdown-steps 1"
if [ "$LOCAL_RANK" = "0" ]; then
  exec ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --cache-control none -k regex:k_round -c 4 --csv \
      --log-file gpurun_out/${TAG}_ncu_round_n${N}.csv python $ARGS
else
  exec python $ARGS
fi
