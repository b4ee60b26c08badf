# r01g, 2 GPUs: parity incl. the host-DRAM tier, multi-rank parity (host tier case), DLRM host-tier bench (W=1)
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf 2>&1 | grep -E "^E  .{0,160}|FAILED|passed|failed" | head -20
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -rf -k "fused-early and not ce" 2>&1 | grep -E "FAILED|passed|failed"
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
print('$2', round(d['value']/1e6,3), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],3) for k,v in d['stages'].items()}, json.dumps(d.get('host_tier')))"; }
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --tables host --variant e --steps 20 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/host_e.log 2>&1; summ gpurun_out/host_e.log host_E
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --tables host --steps 20 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/host_et.log 2>&1; summ gpurun_out/host_et.log host_ET
tail -3 gpurun_out/host_e.log | cut -c1-300
