# ncu --set full of the route and occurrence-sort kernels (DLRM W=1 E variant)
export CUDA_VISIBLE_DEVICES=0
A="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare --variant e"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_radix_scatter|k_radix_hist|k_mark|k_emit|k_inverse|k_expand|k_sched_prep" \
  -s 20 -c 14 -o gpurun_out/prof_route -f python bench.py $A > gpurun_out/prof_route.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_route.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size > gpurun_out/prof_route_summary.csv
