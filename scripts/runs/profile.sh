# Default bench (driver-like) -> ncu launch lists (E+T, E) -> ncu --set full of the row kernels
export CUDA_VISIBLE_DEVICES=0
timeout 900 python bench.py > gpurun_out/prof_bench_default.json 2> gpurun_out/prof_bench_default.err; echo "bench rc=$?"
A="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_launches_et.csv \
  python bench.py $A > gpurun_out/prof_ncu_et.log 2>&1; echo "ncu et rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_launches_e.csv \
  python bench.py --variant e $A > gpurun_out/prof_ncu_e.log 2>&1; echo "ncu e rc=$?"
timeout 1800 ncu --set full --import-source on --clock-control none -k regex:"k_segsum_range|k_segsum_fix|k_pool_stream|k_gather|k_refresh" \
  -s 12 -c 10 -o gpurun_out/prof_full -f python bench.py $A > gpurun_out/prof_ncu_full.log 2>&1; echo "ncu full rc=$?"
rm -f gpurun_out/ncu_traffic.json
python scripts/ncu_traffic.py gpurun_out/prof_full.ncu-rep dlrm/W1/N1 --out gpurun_out/ncu_traffic.json
python scripts/launch_table.py gpurun_out/prof_launches_et.csv > gpurun_out/prof_launches_et.md
python scripts/launch_table.py gpurun_out/prof_launches_e.csv > gpurun_out/prof_launches_e.md
ncu -i gpurun_out/prof_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/prof_full_summary.csv
python scripts/bsum.py gpurun_out/prof_bench_default.json
