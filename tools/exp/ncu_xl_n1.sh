# round-2 ncu evidence of the n=1 bench command (GPT-2 XL): launch list + --set full of K5 and K4a
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_plain.json 2>&1; tail -c 300 gpurun_out/b_plain.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_xl_n1b.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --breakdown-steps 1 > /dev/null 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_adamw_outer|k_sqnorm" --launch-skip 6 --launch-count 2 \
  -f -o gpurun_out/r02_k5_xl python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --breakdown-steps 1 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/r02_k5_xl.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,launch__registers_per_thread,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active > gpurun_out/r02_k5_xl.csv 2>&1; cut -c1-300 gpurun_out/r02_k5_xl.csv
