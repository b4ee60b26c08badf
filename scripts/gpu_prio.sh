# lane priorities (dense,comm,emb; aux = 0): W=1 and W=2
for P in "-2,-1,0" "-2,-1,-1" "-3,-2,-1"; do
NEST_LANE_PRIORITIES=$P CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 60 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/pr1.log 2>&1
NEST_LANE_PRIORITIES=$P timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port $((29600 + RANDOM % 300)) bench.py --gpus 2 --steps 60 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/pr2.log 2>&1
python -c "
import json
for f in ('gpurun_out/pr1.log','gpurun_out/pr2.log'):
    l=[x for x in open(f) if x.startswith('{')][-1]; d=json.loads(l)
    print('prio=$P W=%d'%d['n_gpus'], round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],3) for k,v in d['stages'].items() if k in ('pool','tower','segsum','grad_a2a','update','emb_a2a')})"
done
