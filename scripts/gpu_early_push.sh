# multi-GPU parity (all transports, early push modes) + W=2 bench per early-push mode
for E in ce sm; do NEST_EARLY_PUSH=$E timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "fused-early" 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "not fused-early" 2>&1 | tail -1
for E in ce sm 0; do
NEST_EARLY_PUSH=$E timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port $((29600 + RANDOM % 300)) bench.py --gpus 2 --no-cpu-baseline --no-e2e > gpurun_out/ep_$E.log 2>&1; echo "early=$E rc=$?"
python -c "
import json; l=[x for x in open('gpurun_out/ep_$E.log') if x.startswith('{')][-1]; d=json.loads(l)
print('early=$E', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms', {k: round(v['ms_per_step'],3) for k,v in d['stages'].items()})
print('  N2', json.dumps(d['fwp']['with_tower'].get('N2')), 'emb_only', round(d['embedding_only']['ms_per_step'],3))"
done
