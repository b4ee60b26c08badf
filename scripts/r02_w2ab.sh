T="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
A="--gpus 2 --no-cpu-baseline --no-e2e --steps 30"
p=29600
for r in 1 2; do
for ap in 0 -5; do
for sg in chunks range; do
  p=$((p+1))
  NEST_AUX_PRIORITY=$ap NEST_SEGSUM=$sg timeout 600 $T --master-port $p bench.py $A > gpurun_out/w2ab_ap${ap}_${sg}_r$r.json 2>/dev/null
done; done; done
python scripts/bsum.py gpurun_out/w2ab_*.json
