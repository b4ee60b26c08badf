# r01g final: parity, default bench (driver-like), launch lists (E+T and E), ncu --set full of the row kernels
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf 2>&1 | grep -E "^E  .{0,160}|FAILED|passed|failed" | head -20
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/fin_bench.log 2>&1; tail -c 200 gpurun_out/fin_bench.log
ARGS="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_et.csv python bench.py $ARGS > gpurun_out/fin_ncu_et.log 2>&1; echo rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_e.csv python bench.py --variant e $ARGS > gpurun_out/fin_ncu_e.log 2>&1; echo rc=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_seg|k_pool|k_gather|k_refresh" -s 10 -c 10 \
  -o gpurun_out/fin_full -f python bench.py $ARGS > gpurun_out/fin_ncu_full.log 2>&1; echo rc=$?
