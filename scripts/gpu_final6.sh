# r01g final validation, 4-GPU box: full -m gpu suite (parity, multi-rank W=2 all transports + W=4), smoke, default bench W=1
timeout 2700 python -m pytest tests -m gpu -q -rf 2>&1 | grep -E "FAILED|passed|failed"
CUDA_VISIBLE_DEVICES=0 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/g6_w1.log 2>&1; echo "w1 rc=$?"
python -c "
import json; l=[x for x in open('gpurun_out/g6_w1.log') if x.startswith('{')][-1]; d=json.loads(l)
print('W=1', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms; e2e', round(d['e2e']['value']/1e6,2), 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3), 'clk', d['clocks'], 'E', round(d['embedding_only']['ms_per_step'],3), 'cpu', d['cpu_baseline']['value'], 'launches', d['gpu_launches'])"
