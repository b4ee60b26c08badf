# SGD vs row-wise AdaGrad, W=1 and W=2 (default bench otherwise)
for O in sgd rowwise_adagrad; do
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e --optimizer $O > gpurun_out/opt1_$O.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) \
  bench.py --gpus 2 --steps 50 --no-cpu-baseline --no-e2e --optimizer $O > gpurun_out/opt2_$O.log 2>&1
for W in 1 2; do python -c "
import json; l=[x for x in open('gpurun_out/opt${W}_$O.log') if x.startswith('{')][-1]; d=json.loads(l)
print('$O W=%d'%d['n_gpus'], round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'emb_only', round(d['embedding_only']['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['stages'].items() if k in ('segsum','update','grad_a2a')}, 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3))"; done
done
