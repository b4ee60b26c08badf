# GPU parity suite + smoke + W=1 default bench (x2)
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for rep in 1 2; do
timeout 600 python bench.py --steps 60 --no-cpu-baseline --no-e2e > gpurun_out/q_$rep.log 2>&1
python -c "
import json; l=[x for x in open('gpurun_out/q_$rep.log') if x.startswith('{')][-1]; d=json.loads(l)
print('rep=$rep', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'emb_only', round(d['embedding_only']['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
done
