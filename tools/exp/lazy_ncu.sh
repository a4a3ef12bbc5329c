# sharded lazy step in VirtualGroups on one GPU: live timing, then ncu --set full of its two kernels
for N in 2 4; do
timeout 300 python tools/lazy_profile.py --n $N
NS=$((2*N))
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p2p_reduce|k_lazy_adamw_push" --launch-skip $NS --launch-count $NS \
  -f -o gpurun_out/lazy_n$N python tools/lazy_profile.py --n $N --steps 1 > gpurun_out/lazy_ncu_n$N.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/lazy_n$N.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,launch__registers_per_thread,launch__grid_size > gpurun_out/lazy_n$N.csv 2>&1
cut -c1-250 gpurun_out/lazy_n$N.csv | head -12
done
