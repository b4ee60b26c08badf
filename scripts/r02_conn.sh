export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --no-e2e --steps 30"
for r in 1 2; do for c in 8 32; do
  CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 300 python bench.py $A > gpurun_out/conn${c}_r$r.json 2>/dev/null
done; done
python scripts/bsum.py gpurun_out/conn*_r*.json
