# 2-GPU box: all GPU tests, default bench at W=1 and W=2
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/bench_w1.log 2>&1; echo "w1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --gpus 2 > gpurun_out/bench_w2.log 2>&1; echo "w2 rc=$?"
for f in gpurun_out/bench_w1.log gpurun_out/bench_w2.log; do
python -c "
import json; l=[x for x in open('$f') if x.startswith('{')][-1]; d=json.loads(l)
print('$f', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms; e2e', round(d['e2e']['value']/1e6,2), 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3), 'traffic', d['roofline']['traffic'])
print('  with_tower', json.dumps(d['fwp']['with_tower']))
print('  a2a', json.dumps({k:v for k,v in (d['a2a'] or {}).items() if k!='with_tower'}))"
done
