export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "zero_copy" 2>&1 | tail -3
NEST_ZERO_COPY=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bench_path or p1 or refresh or host" 2>&1 | tail -3
A="--no-cpu-baseline --no-e2e --steps 30"
for r in 1 2; do for z in 0 1; do
  NEST_ZERO_COPY=$z timeout 300 python bench.py $A > gpurun_out/zc${z}_r$r.json 2>/dev/null
done; done
python scripts/bsum.py gpurun_out/zc*_r*.json
