# r01g, 2 GPUs: gather skips the pending update's keys (refresh supplies them): parity, multi-rank, W=1/W=2 + host-tier bench
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf 2>&1 | grep -E "^E  .{0,160}|FAILED|passed|failed" | head -20
timeout 1800 python -m pytest tests/test_gpu_multi.py -q -rf 2>&1 | grep -E "FAILED|passed|failed"
CUDA_VISIBLE_DEVICES=0 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
e=d.get('embedding_only') or {}
print('$2', round(d['value']/1e6,3), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'E', round(e.get('ms_per_step',0),3), {k: round(v['ms_per_step'],3) for k,v in d['stages'].items()}, 'frac', round(d['roofline']['frac'],3), json.dumps(d.get('host_tier')))"; }
for rep in 1 2; do
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/sk_w1_$rep.log 2>&1; summ gpurun_out/sk_w1_$rep.log w1_$rep
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29741 \
  bench.py --gpus 2 --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/sk_w2.log 2>&1; summ gpurun_out/sk_w2.log w2
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --tables host --variant e --steps 20 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/sk_host_e.log 2>&1; summ gpurun_out/sk_host_e.log host_E
