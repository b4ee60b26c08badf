export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --no-e2e --steps 30 --no-fwp-compare"
for g in 0 40 56 72; do
for N in 1 2; do
for pf in 2 3; do
  NEST_GREEN_SMS=$g NEST_TOWER_SM_RESERVE=$([ $g = 0 ] && echo 24 || echo $g) NEST_PF=$pf \
    timeout 300 python bench.py $A --micro-batches $N > gpurun_out/gr${g}_N${N}_pf${pf}.json 2>gpurun_out/gr${g}_N${N}_pf${pf}.err
done; done; done
python scripts/bsum.py gpurun_out/gr*_N*_pf*.json
grep -l Traceback gpurun_out/gr*.err | head; tail -3 $(ls gpurun_out/gr*.err | head -1)
