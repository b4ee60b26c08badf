# W=2: grads by SM remote stores vs local + copy engine
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "gradce" 2>&1 | tail -1
for rep in 1 2; do for G in sm ce; do
NEST_GRAD_PUSH=$G timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port $((29600 + RANDOM % 300)) bench.py --gpus 2 --steps 80 --no-cpu-baseline --no-e2e > gpurun_out/gc_$G.log 2>&1
python -c "
import json; l=[x for x in open('gpurun_out/gc_$G.log') if x.startswith('{')][-1]; d=json.loads(l)
print('rep=$rep grad=$G', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'emb_only', round(d['embedding_only']['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['stages'].items() if k in ('segsum','grad_a2a','update','pool','tower')})"
done; done
