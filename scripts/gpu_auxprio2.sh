# r01g: DBP lookahead stream priority with the final kernels, W=4 and W=2 (A/B/A/B)
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
print('$2', round(d['value']/1e6,3), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'])"; }
run() { W=$1; tag=$2; shift 2; env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port $((29800 + RANDOM % 100)) \
  bench.py --gpus $W --steps 50 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/ap2_$tag.log 2>&1; summ gpurun_out/ap2_$tag.log $tag; }
for rep in 1 2; do
run 4 w4_p0_$rep NEST_AUX_PRIORITY=0
run 4 w4_p1_$rep NEST_AUX_PRIORITY=-1
run 4 w4_p3_$rep NEST_AUX_PRIORITY=-3
run 2 w2_p0_$rep NEST_AUX_PRIORITY=0
run 2 w2_p3_$rep NEST_AUX_PRIORITY=-3
done
