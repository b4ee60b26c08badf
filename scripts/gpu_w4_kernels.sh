# r01g, 4 GPUs: W=4 bench, r01 pool/segment-sum kernels vs the streaming/range ones (A/B/A/B)
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
e=d.get('embedding_only') or {}
print('$2', round(d['value']/1e6,3), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'E', round(e.get('ms_per_step',0),3), {k: round(v['ms_per_step'],3) for k,v in d['stages'].items()})"; }
run() { W=$1; tag=$2; shift 2; env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port $((29800 + RANDOM % 100)) \
  bench.py --gpus $W --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/k4_$tag.log 2>&1; summ gpurun_out/k4_$tag.log $tag; }
run 4 old1 NEST_SEGSUM=chunks NEST_POOL=bag
run 4 new1 NEST_SEGSUM=range
run 4 old2 NEST_SEGSUM=chunks NEST_POOL=bag
run 4 new2 NEST_SEGSUM=range
