# bf16 hand-off: parity tests + W=1 bench A/B
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for rep in 1 2; do for P in 1 0; do
NEST_BENCH_POOLED_BF16=$P timeout 600 python bench.py --steps 60 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/bf_$P.log 2>&1
python -c "
import json; l=[x for x in open('gpurun_out/bf_$P.log') if x.startswith('{')][-1]; d=json.loads(l)
print('rep=$rep bf16=$P', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],3) for k,v in d['stages'].items() if k in ('pool','tower','segsum','tower_dw')})"
done; done
