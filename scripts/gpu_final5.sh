# r01g final (tower SM reserve 0), 4-GPU box: full -m gpu suite, multi-rank parity, default bench W=1, 2, 4
timeout 2400 python -m pytest tests -m gpu -q -rf 2>&1 | grep -E "FAILED|passed|failed"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/g5_w1.log 2>&1; echo "w1 rc=$?"
for W in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port $((29870 + W)) \
  bench.py --gpus $W > gpurun_out/g5_w$W.log 2>&1; echo "w$W rc=$?"
done
for W in 1 2 4; do
python -c "
import json; l=[x for x in open('gpurun_out/g5_w$W.log') if x.startswith('{')][-1]; d=json.loads(l)
print('W=$W', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms; e2e', round(d['e2e']['value']/1e6,2), 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'], 'emb_only', round(d['embedding_only']['samples_per_s']/1e6,2), round(d['embedding_only']['ms_per_step'],3))
w=d['fwp']['with_tower'].get('N2'); print('   N2', w and (round(w['samples_per_s']/1e6,2), round(w['ms_per_step'],3), round(w.get('a2a_exposed_ratio') or 0,3)), 'a2a', d['a2a'] and {k: round(v,3) for k,v in d['a2a'].items() if isinstance(v,float)})"
done
