export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --no-e2e --steps 30 --no-fwp-compare"
for r in 1 2; do
for sr in 0 24 48; do
  NEST_TOWER_SM_RESERVE=$sr timeout 300 python bench.py $A > gpurun_out/smr${sr}_r$r.json 2>/dev/null
done
for lp in "-2,-1,0" "-2,-1,-2" "-1,-1,-1"; do
  NEST_LANE_PRIORITIES=$lp timeout 300 python bench.py $A > gpurun_out/lp${lp}_r$r.json 2>/dev/null
done
done
python scripts/bsum.py gpurun_out/smr*_r*.json gpurun_out/lp*_r*.json
