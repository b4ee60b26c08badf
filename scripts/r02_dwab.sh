export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --no-e2e --steps 30"
for r in 1 2; do
for da in 0 1; do
for ap in 0 -5; do
  NEST_AUX_PRIORITY=$ap NEST_TOWER_DW_AFTER_BWD=$da timeout 300 python bench.py $A > gpurun_out/dw${da}_ap${ap}_r$r.json 2>/dev/null
done; done; done
python scripts/bsum.py gpurun_out/dw*_r*.json
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "tower or bench_path" 2>&1 | tail -2
NEST_TOWER_DW_AFTER_BWD=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "tower" 2>&1 | tail -2
