# r01g: k_emit segment search hoisted per word -- parity (W=1, W=2), E bench, launch list
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf 2>&1 | grep -E "^E  .{0,200}|FAILED|passed|failed" | head -20
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -rf -k "2-fused-early]" 2>&1 | grep -E "FAILED|passed|failed"
export CUDA_VISIBLE_DEVICES=0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/em_launches_e.csv \
  python bench.py --variant e --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare > gpurun_out/em_ncu_e.log 2>&1; echo rc=$?
