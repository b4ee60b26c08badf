export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --no-e2e --steps 30"
for r in 1 2; do
for ap in 0 -1 -3 -5; do
  NEST_AUX_PRIORITY=$ap timeout 300 python bench.py $A > gpurun_out/ap${ap}_r$r.json 2>/dev/null
done
done
python scripts/bsum.py gpurun_out/ap*_r*.json
