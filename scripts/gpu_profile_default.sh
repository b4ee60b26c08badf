# Default bench (W=1 DLRM E+T) -> launch list -> ncu --set full of the row kernels
export CUDA_VISIBLE_DEVICES=0
ARGS="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare"
timeout 600 python bench.py > gpurun_out/bench_default.json.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv \
  python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1 || exit 2
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_seg|k_pool|k_gather|k_refresh" \
  -s 10 -c 10 -o gpurun_out/full_default -f python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1 || exit 3
echo done
