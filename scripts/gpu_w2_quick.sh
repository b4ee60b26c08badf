# 2-GPU: GPU parity (1 GPU) + multi-rank parity + W=1 / W=2 bench
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 60 --no-cpu-baseline --no-e2e > gpurun_out/wq_w1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29712 \
  bench.py --gpus 2 --steps 60 --no-cpu-baseline --no-e2e > gpurun_out/wq_w2.log 2>&1
for W in 1 2; do
python -c "
import json; l=[x for x in open('gpurun_out/wq_w$W.log') if x.startswith('{')][-1]; d=json.loads(l)
print('W=$W', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'emb_only', round(d['embedding_only']['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
done
