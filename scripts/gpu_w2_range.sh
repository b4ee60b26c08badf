# r01g, 2 GPUs: parity (1 GPU), multi-rank parity (every transport), W=2 bench new vs r01 kernels
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -rf 2>&1 | grep -E "FAILED|passed|failed"
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
e=d['embedding_only']
print('$2', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'E', round(e['ms_per_step'],3), {k: round(v,3) for k,v in e['stage_ms_per_step'].items()}, 'frac', round(d['roofline']['frac'],3))"; }
for rep in 1 2; do
NEST_POOL=bag NEST_SEGSUM=chunks timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2971$rep \
  bench.py --gpus 2 --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/w2r_old_$rep.log 2>&1; summ gpurun_out/w2r_old_$rep.log old$rep
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2972$rep \
  bench.py --gpus 2 --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/w2r_new_$rep.log 2>&1; summ gpurun_out/w2r_new_$rep.log new$rep
done
