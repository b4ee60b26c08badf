# default bench at W=1, 2, 4 (one box); summary lines at the end
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/scale_w1.log 2>&1; echo "w1 rc=$?"
for W in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2953$W \
  bench.py --gpus $W > gpurun_out/scale_w$W.log 2>&1; echo "w$W rc=$?"
done
for W in 1 2 4; do
python -c "
import json; l=[x for x in open('gpurun_out/scale_w$W.log') if x.startswith('{')][-1]; d=json.loads(l)
print('W=$W', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms; e2e', round(d['e2e']['value']/1e6,2), 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3), 'clk', d['clocks'])
print('  with_tower', json.dumps(d['fwp']['with_tower']))
print('  emb_only', json.dumps({k:v for k,v in (d['embedding_only'] or {}).items() if k!='stage_ms_per_step'}))
print('  a2a', json.dumps({k:v for k,v in (d['a2a'] or {}).items() if k!='with_tower'}))"
done
