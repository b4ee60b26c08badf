# default bench -> launch list -> ncu --set full of the route / sort / pool kernels
export CUDA_VISIBLE_DEVICES=0
ARGS="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare"
timeout 600 python bench.py $ARGS > gpurun_out/pr_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv \
  python bench.py $ARGS > gpurun_out/ncu_launch2.log 2>&1 || exit 2
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_inverse|k_mark|k_radix|k_emit|k_pool|k_expand" \
  -s 14 -c 9 -o gpurun_out/full_route -f python bench.py $ARGS > gpurun_out/ncu_full2.log 2>&1 || exit 3
echo done
