# r01g, 4 GPUs: which of the new kernels slows W=4 (segment-sum or pool), and the aux stream priority
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
e=d.get('embedding_only') or {}
print('$2', round(d['value']/1e6,3), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'E', round(e.get('ms_per_step',0),3))"; }
run() { W=$1; tag=$2; shift 2; env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port $((29800 + RANDOM % 100)) \
  bench.py --gpus $W --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/sp_$tag.log 2>&1; summ gpurun_out/sp_$tag.log $tag; }
for rep in 1 2; do
run 4 segchunks_poolstream_$rep NEST_SEGSUM=chunks
run 4 segrange_poolbag_$rep NEST_POOL=bag
run 4 old_auxp3_$rep NEST_SEGSUM=chunks NEST_POOL=bag NEST_AUX_PRIORITY=-3
run 4 new_auxp3_$rep NEST_AUX_PRIORITY=-3
done
