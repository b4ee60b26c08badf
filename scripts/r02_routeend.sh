export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --no-e2e --steps 30"
for r in 1 2 3; do for m in after_grad before_grad; do
  NEST_ROUTE_END=$m timeout 300 python bench.py $A > gpurun_out/re_${m}_r$r.json 2>/dev/null
done; done
python scripts/bsum.py gpurun_out/re_*_r*.json
