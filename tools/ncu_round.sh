# usage (1-GPU gpurun box): bash tools/ncu_round.sh TAG
# launch list of the fused XL step + ncu --set full of the streaming kernels (GPT-2 small)
TAG=${1:-r01}
set -x
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/pre_launch.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_xl_fused.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
python bench.py --config small --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/pre_small.json 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_adamw|k_sqnorm|k_outer_update" -c 8 \
    -o gpurun_out/${TAG}_ncu_small -f python bench.py --config small --steps 2 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"^k_adamw$|^k_outer_update$" -c 2 \
    -o gpurun_out/${TAG}_ncu_small_k4b -f python bench.py --config small --steps 2 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/ncu_full_k4b.log 2>&1
ls -la gpurun_out
