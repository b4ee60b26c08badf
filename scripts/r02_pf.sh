export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --no-e2e --steps 30"
for r in 1 2; do
for pf in 0 1 2 3; do
  NEST_PF=$pf timeout 300 python bench.py $A > gpurun_out/pf${pf}_r$r.json 2>/dev/null
done
done
python scripts/bsum.py gpurun_out/pf*_r*.json
