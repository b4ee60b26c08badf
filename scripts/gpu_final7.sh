# r01g last check (1 GPU): -m gpu suite, smoke, default bench (driver-like)
export CUDA_VISIBLE_DEVICES=0
timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | grep -E "FAILED|passed|failed"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/g7_w1.log 2>&1; echo "w1 rc=$?"
python -c "
import json; l=[x for x in open('gpurun_out/g7_w1.log') if x.startswith('{')][-1]; d=json.loads(l)
print('W=1', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms; e2e', round(d['e2e']['value']/1e6,2), 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3), 'clk', d['clocks'], 'E', round(d['embedding_only']['ms_per_step'],3), round(d['embedding_only']['roofline']['frac'],3))"
