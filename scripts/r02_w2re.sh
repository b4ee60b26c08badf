T="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
A="--gpus 2 --no-cpu-baseline --no-e2e --steps 30 --variant e --no-fwp-compare"
p=29850
for r in 1 2; do for m in after_grad before_grad; do
  p=$((p+1)); NEST_ROUTE_END=$m timeout 600 $T --master-port $p bench.py $A > gpurun_out/w2re_${m}_r$r.json 2>/dev/null
done; done
python scripts/bsum.py gpurun_out/w2re_*_r*.json
