export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --no-e2e --steps 30"
for r in 1 2; do for rx in classic onesweep; do
  NEST_RADIX=$rx timeout 300 python bench.py $A > gpurun_out/rx_${rx}_r$r.json 2>/dev/null
done; done
python scripts/bsum.py gpurun_out/rx_*_r*.json
NEST_RADIX=onesweep timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "p1 or route or cluster" 2>&1 | tail -2
