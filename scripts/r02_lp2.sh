export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --no-e2e --steps 30 --no-fwp-compare"
for r in 1 2 3; do
for lp in "-2,-1,0" "-2,-1,-4" "-3,-1,-4"; do
  NEST_LANE_PRIORITIES=$lp timeout 300 python bench.py $A > gpurun_out/lp2${lp}_r$r.json 2>/dev/null
done; done
python scripts/bsum.py gpurun_out/lp2*_r*.json
